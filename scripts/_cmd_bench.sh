export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python bench.py $BENCH_ARGS > gpurun_out/bench_r01h.json 2> gpurun_out/bench_r01h.err; echo "bench rc=$?"
python - <<'P'
import json; d=json.load(open("gpurun_out/bench_r01h.json"))
print("value", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], "kernel_ms", d["roofline"]["kernel_ms"], "e2e", d["e2e"]["value"], d["clocks"])
for k in ("ipg","ipg_cfg2","ipg_cfg4"):
    if k in d: print(k, d[k]["ms_per_iter"], d[k].get("roofline_model",{}).get("frac"))
print("cfg3", d.get("cfg3",{}).get("ms_per_projection"))
P
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r01h_ref.json 2>gpurun_out/bench_r01h_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_r01h_ref.json
