"""Per-kernel table from one ncu --set full report holding several launches (operator kernels):
duration, DRAM bytes, achieved DRAM GB/s, issue / LSU utilisation, shared-memory bank conflicts.

    python scripts/summarize_ncu_multi.py <report.ncu-rep> <out.txt> [command line]
"""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def num(r, key):
    if key not in col:
        return float("nan")
    try:
        return float(r[col[key]].replace(",", ""))
    except ValueError:
        return float("nan")


def scaled(r, key, to):
    v, u = num(r, key), units[col[key]] if key in col else ""
    f = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9}.get(u, 1.0)
    return v * f / to


def top_stalls(r, k=3):
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    xs = []
    for h, i in col.items():
        if h.startswith(pre) and h.endswith(suf):
            try:
                xs.append((float(r[i].replace(",", "")), h[len(pre):-len(suf)]))
            except ValueError:
                pass
    return sorted(xs, reverse=True)[:k]


with open(out, "w") as fh:
    fh.write(f"{cmd}\n(ncu --set full: cold caches, serialised launches)\n\n")
    fh.write(f"{'kernel':44s} {'ms':>8s} {'dram MB':>9s} {'GB/s':>7s} {'issue%':>7s} {'lsu%':>6s} "
             f"{'alu%':>6s} {'fma%':>6s} {'L2hit%':>7s} {'smem confl/req':>14s} {'warps%':>7s}\n")
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("cbb::", "")
        t = scaled(r, "gpu__time_duration.sum", 1e-3)
        b = scaled(r, "dram__bytes_read.sum", 1e6) + scaled(r, "dram__bytes_write.sum", 1e6)
        wf = num(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        rq = num(r, "smsp__inst_executed_op_shared_ld.sum") + num(r, "smsp__inst_executed_op_shared_st.sum")
        fh.write(f"{name[:44]:44s} {t:8.3f} {b:9.1f} {b / t if t else 0:7.0f} "
                 f"{num(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):7.1f} "
                 f"{num(r, 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active'):6.1f} "
                 f"{num(r, 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):6.1f} "
                 f"{num(r, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):6.1f} "
                 f"{num(r, 'lts__t_sector_hit_rate.pct'):7.1f} "
                 f"{(wf / rq if rq else float('nan')):14.2f} "
                 f"{num(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):7.1f}  "
                 + " ".join(f"{k}={v:.2f}" for v, k in top_stalls(r)) + "\n")
print(open(out).read())
