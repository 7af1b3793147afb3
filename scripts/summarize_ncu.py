"""Summaries committed under profiles/ from the two ncu passes of the profiling recipe.

    python scripts/summarize_ncu.py launches <launches.csv> <out.txt> [command line]
    python scripts/summarize_ncu.py full <report.ncu-rep> <out.txt> <traffic.json> [command]

``launches``: per-kernel totals of gpu__time_duration.sum (cold-cache, serialised launches:
compare shares, not absolute times).  ``full``: key metrics, stall breakdown and the DRAM
traffic of the captured matched-filter launch; the traffic JSON feeds bench.py's roofline.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path, out, cmd):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rd:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r["Metric Unit"], 1e-6)
        tot[name] += v * scale
        cnt[name] += 1
    total = sum(tot.values())
    with open(out, "w") as fh:
        fh.write(f"{cmd}\n(cold-cache, serialised launches: compare SHARES, not absolute times)\n\n")
        for name, ms in sorted(tot.items(), key=lambda x: -x[1]):
            fh.write(f"{ms:10.3f} ms {100 * ms / total:6.2f}%  launches={cnt[name]:4d}  "
                     f"mean={1e3 * ms / cnt[name]:9.1f} us  {name[:70]}\n")
    print(open(out).read())


KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
]


def full(rep, out, traffic_json, cmd):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    name = d.get("Kernel Name", ("?", ""))[0]
    with open(out, "w") as fh:
        fh.write(f"{cmd}\nkernel: {name}\n\n")
        for k in KEYS:
            if k in d:
                fh.write(f"{k:90s} {d[k][0]:>14} {d[k][1]}\n")
        stalls = [(k, d[k][0]) for k in hdr
                  if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio")]
        stalls.sort(key=lambda kv: -float(kv[1].replace(",", "") or 0))
        fh.write("\nstalls per issued instruction (top 8):\n")
        for k, v in stalls[:8]:
            fh.write(f"  {k:88s} {v}\n")
    print(open(out).read())

    def num(key):
        v, u = d[key]
        v = float(v.replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    t = {"kernel": name, "report": rep.split("/")[-1],
         "dram_bytes_read": num("dram__bytes_read.sum"),
         "dram_bytes_write": num("dram__bytes_write.sum")}
    t["dram_bytes_per_launch"] = t["dram_bytes_read"] + t["dram_bytes_write"]
    t["tensor_pipe_active_pct"] = num(
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    t["issue_active_pct"] = num("smsp__issue_active.avg.pct_of_peak_sustained_active")
    with open(traffic_json, "w") as fh:
        json.dump(t, fh, indent=1)
    print(t)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else "")
