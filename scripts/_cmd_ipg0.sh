export PYTHONPATH=.
mkdir -p gpurun_out
python scripts/probe_ipg0.py 4 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ipg0_launches.csv python scripts/probe_ipg0.py 3 > gpurun_out/ncu_ipg0.log 2>&1
python scripts/summarize_ncu.py launches gpurun_out/ipg0_launches.csv gpurun_out/ipg0_launches.txt "probe_ipg0 (one cfg0 solve)"
head -30 gpurun_out/ipg0_launches.txt
