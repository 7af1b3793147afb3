export PYTHONPATH=.
mkdir -p gpurun_out
for c in cfg2 cfg4; do
  timeout 600 python scripts/probe_ipg.py $c 6 2>&1 | grep -v Warn | tail -10
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ipg_launches_$c.csv python scripts/probe_ipg.py $c 3 > gpurun_out/ncu_ipg_$c.log 2>&1
  echo "ncu $c rc=$?"
  python scripts/summarize_ncu.py launches gpurun_out/ipg_launches_$c.csv gpurun_out/ipg_launches_$c.txt "probe_ipg $c 3"
  head -25 gpurun_out/ipg_launches_$c.txt
done
