export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py -x -q > gpurun_out/r02_prune_pytest.log 2>&1; echo "pytest prune rc=$?"; tail -30 gpurun_out/r02_prune_pytest.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_all_pytest.log 2>&1; echo "pytest all rc=$?"; tail -3 gpurun_out/r02_all_pytest.log
timeout 900 python bench.py --skip-cfg3 > gpurun_out/r02_prune_bench.json 2> gpurun_out/r02_prune_bench.err; echo "bench rc=$?"
tail -5 gpurun_out/r02_prune_bench.err
python - <<'P'
import json; d=json.load(open("gpurun_out/r02_prune_bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], "kernel_ms", d["roofline"]["kernel_ms"], "e2e", d["e2e"]["value"], d["clocks"])
for k in ("ipg","ipg_cfg2","ipg_cfg4"):
    if k in d: print(k, d[k].get("ms_per_iter"), d[k].get("roofline_model",{}).get("frac"), d[k].get("error"), d[k].get("iterations"), d[k].get("final_fidelity"))
P
