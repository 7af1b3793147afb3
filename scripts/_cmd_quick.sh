export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python scripts/probe_cfg1.py 2>&1 | tail -3
timeout 300 python bench.py --skip-cfg3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python - <<'P'
import json; d=json.load(open("gpurun_out/bench_q.json"))
print("value", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], "kernel_ms", d["roofline"]["kernel_ms"], "e2e", d["e2e"]["value"])
for k in ("ipg","ipg_cfg2","ipg_cfg4"):
    if k in d: print(k, d[k]["ms_per_iter"], d[k].get("roofline_model",{}).get("frac"))
P
