export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_op_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_op_pytest.log
timeout 900 python bench.py --skip-cfg3 --skip-cpu-reference > gpurun_out/r02_op_bench.json 2> gpurun_out/r02_op_bench.err; echo "bench rc=$?"
python - <<'P'
import json; d=json.load(open("gpurun_out/r02_op_bench.json"))
print("value", d["value"], "kernel_ms", d["roofline"]["kernel_ms"])
for k in ("ipg","ipg_cfg2","ipg_cfg4"):
    x = d.get(k, {}); print(k, x.get("ms_per_iter"), repr(x.get("final_fidelity")), x.get("error"), "unsharded", (x.get("unsharded") or {}).get("ms_per_iter"), repr((x.get("unsharded") or {}).get("final_fidelity")))
    if "unsharded" in x: print("  operator", json.dumps(x["unsharded"].get("operator")))
print(json.dumps(d["parity"])[:600])
P
