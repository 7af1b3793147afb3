export PYTHONPATH=.
mkdir -p gpurun_out
R=${R:-r02a}
timeout 1200 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_$R.err
python - <<P
import json; d=json.load(open("gpurun_out/bench_$R.json"))
print("value", d["value"], "frac", d["roofline"]["frac"], "kernel_ms", d["roofline"]["kernel_ms"], "e2e", d["e2e"]["value"], "pageable ms", d["e2e"].get("pageable_ms_per_step"), d["clocks"])
print("parity", json.dumps(d.get("parity"))[:1500])
for k in ("ipg","ipg_cfg2","ipg_cfg4"):
    x = d.get(k, {}); print(k, x.get("ms_per_iter"), x.get("roofline_model",{}).get("frac"), x.get("error"), (x.get("tile_pruning") or {}).get("mean_listed_fraction"), "unsharded", (x.get("unsharded") or {}).get("ms_per_iter"))
    if "unsharded" in x: print("  operator", json.dumps(x["unsharded"].get("operator"))[:600])
print("cfg3", d.get("cfg3",{}).get("ms_per_projection"), d.get("cfg3",{}).get("error"))
cb = d.get("cpu_baseline", {}); print("cpu", cb.get("value"), json.dumps(cb.get("host")), json.dumps(cb.get("reference_legs"))[:800])
P
