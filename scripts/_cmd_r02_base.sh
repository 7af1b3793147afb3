export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_base_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_base_pytest.log
timeout 900 python bench.py > gpurun_out/r02_base_bench.json 2> gpurun_out/r02_base_bench.err; echo "bench rc=$?"
python - <<'P'
import json; d=json.load(open("gpurun_out/r02_base_bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], "kernel_ms", d["roofline"]["kernel_ms"], "e2e", d["e2e"]["value"], d["clocks"])
for k in ("ipg","ipg_cfg2","ipg_cfg4"):
    if k in d: print(k, d[k].get("ms_per_iter"), d[k].get("roofline_model",{}).get("frac"), d[k].get("error"))
print("cfg3", d.get("cfg3",{}).get("ms_per_projection"))
P
nproc; lscpu | grep -i "model name"; python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A3 blas | head -20
