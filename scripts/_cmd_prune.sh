export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python scripts/probe_prune.py cfg4 > gpurun_out/prune2_cfg4.log 2>&1; echo "cfg4 rc=$?"
timeout 600 python scripts/probe_prune.py cfg2 > gpurun_out/prune2_cfg2.log 2>&1; echo "cfg2 rc=$?"
cat gpurun_out/prune2_cfg4.log gpurun_out/prune2_cfg2.log | grep -v Warn | tail -40
