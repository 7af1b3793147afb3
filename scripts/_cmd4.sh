export PYTHONPATH=.
mkdir -p gpurun_out
python scripts/probe_cfg4.py 20 > gpurun_out/cfg4_20.log 2>&1
PROBE_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python scripts/probe_cfg4.py > gpurun_out/cfg4_ncu.log 2>&1
tail -30 gpurun_out/cfg4_20.log
