export PYTHONPATH=.
mkdir -p gpurun_out
PROBE_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches_split.csv python scripts/probe_cfg4.py > gpurun_out/cfg4_ncu.log 2>&1
python scripts/probe_cfg2.py > /dev/null 2>&1
