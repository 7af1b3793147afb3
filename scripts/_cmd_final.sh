# final validation of a round: GPU tests, smoke, default bench + reference arm
export PYTHONPATH=.
mkdir -p gpurun_out
R=${R:-r02i}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$R.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$R.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${R}_reference.json 2> gpurun_out/bench_${R}_reference.err; echo "ref rc=$?"
python - <<P
import json; d=json.load(open("gpurun_out/bench_$R.json"))
print("value", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], "kernel_ms", d["roofline"]["kernel_ms"], "e2e", d["e2e"]["value"], d["clocks"])
for k in ("ipg","ipg_cfg2","ipg_cfg4"):
    x = d.get(k, {}); print(k, x.get("ms_per_iter"), x.get("error"), "unsharded", (x.get("unsharded") or {}).get("ms_per_iter"), json.dumps(x.get("cpu_model"))[:200])
    if "unsharded" in x: print("  operator", json.dumps({a:(round(b["ms"],3), round(b["frac"],3)) for a,b in x["unsharded"]["operator"].items() if isinstance(b, dict)}))
print("cfg3", d.get("cfg3",{}).get("ms_per_projection"))
print("parity", json.dumps(d["parity"])[:400])
P
