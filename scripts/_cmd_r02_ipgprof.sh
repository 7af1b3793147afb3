export PYTHONPATH=.
mkdir -p gpurun_out
for c in cfg4; do
  timeout 600 python scripts/probe_ipg.py $c 20 2>&1 | grep -v Warn | tail -12
  timeout 900 ncu --graph-profiling node --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --launch-skip 0 --csv --log-file gpurun_out/ipg_launches_$c.csv python scripts/probe_ipg.py $c 6 nograph > gpurun_out/ncu_ipg_$c.log 2>&1
  echo "ncu $c rc=$?"
  python scripts/summarize_ncu.py launches gpurun_out/ipg_launches_$c.csv gpurun_out/ipg_launches_$c.txt "probe_ipg $c 4"
  head -22 gpurun_out/ipg_launches_$c.txt
done
