export PYTHONPATH=.
mkdir -p gpurun_out
timeout 300 python scripts/probe_cfg4.py 3 2>&1 | tail -4
PROBE_PROFILE=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/probe_cfg4.py > gpurun_out/c4_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/summarize_ncu.py launches gpurun_out/c4_launches.csv gpurun_out/c4_launches.txt "cfg4 1 iteration" | head -30
