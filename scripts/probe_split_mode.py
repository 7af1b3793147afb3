"""Split-operand (fp32-accumulated) tcgen05 screen vs the fp16 screen: agreement, oracle parity
on a small coherent case, timings and overflow counts on cfg1 and a cfg4-like coherent case."""
import sys

import numpy as np
import torch

from paper_1810_01967_b200 import device_dictionary, workloads
from paper_1810_01967_b200.projection import overflow_counts, project_device

dev = torch.device("cuda:0")


def kernel_ms(Z, dd, algo, reps=3):
    """matched-filter kernel alone (library CUDA events around the screen)."""
    import ctypes
    from paper_1810_01967_b200 import _lib
    lib = _lib.load()
    lib.cbb_timing_enable(1)
    tot = 0.0
    for _ in range(reps):
        project_device(Z, dd, algo=algo)
        ms = ctypes.c_float(0)
        lib.cbb_timing_last_ms(ctypes.byref(ms))
        tot += ms.value
    lib.cbb_timing_enable(0)
    return tot / reps


def timeit(Z, dd, algo, reps=3):
    out = project_device(Z, dd, algo=algo)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        out = project_device(Z, dd, algo=algo)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps, out


def compare(name, Z, dd, algos=("tcgen05_split", "tcgen05")):
    res = {}
    for a in algos:
        ms, out = timeit(Z, dd, a)
        cnt = overflow_counts(Z.shape[0], Z.shape[1])
        res[a] = out
        kms = kernel_ms(Z, dd, a)
        print(f"{name:10s} {a:14s} {ms:9.3f} ms (screen kernel {kms:8.3f} ms)  "
              f"overflow(exh, warp) {cnt}", flush=True)
    i0 = res[algos[0]][0]
    for a in algos[1:]:
        same = bool(torch.equal(i0, res[a][0]))
        print(f"{name:10s} indices {algos[0]} == {a}: {same}; "
              f"gamma max diff {float((res[a][1] - res[algos[0]][1]).abs().max()):.3g}", flush=True)


which = sys.argv[1:] or ["small", "cfg1", "coh"]
if "small" in which:
    from oracle import projection as orc
    cd, raw = workloads._offres_dictionary(200, 10, 40, 40, 11, dev)
    atoms = cd.atoms_compressed
    rng = np.random.default_rng(0)
    n = 8192
    idx = rng.integers(len(atoms), size=n)
    Z = atoms[idx] * rng.uniform(0.2, 1, size=(n, 1)) + 0.05 * (
        rng.standard_normal((n, 10)) + 1j * rng.standard_normal((n, 10)))
    dd = device_dictionary(atoms, dev)
    ref = orc.project_cone_exact(Z, atoms)
    for a in ("tcgen05", "tcgen05_split", "ffma"):
        got = project_device(torch.from_numpy(Z).to(dev), dd, algo=a)
        gi = got[0].cpu().numpy()
        print(f"small coherent d={len(atoms)} {a:14s} index mismatches vs oracle: "
              f"{int((gi != ref.indices).sum())}  overflow {overflow_counts(n, 10)}", flush=True)
if "cfg1" in which:
    atoms, Z, gen = workloads.make_cfg1()
    dd = device_dictionary(atoms, dev)
    compare("cfg1", torch.from_numpy(Z).to(dev), dd)
if "coh" in which:
    cd, raw = workloads._offres_dictionary(500, 10, 100, 100, 26, dev)
    atoms = cd.atoms_compressed
    del raw
    rng = np.random.default_rng(1)
    n = 1 << 20
    idx = rng.integers(len(atoms), size=n)
    Z = atoms[idx] * rng.uniform(0.5, 1, size=(n, 1)) + 0.1 / np.sqrt(20) * (
        rng.standard_normal((n, 10)) + 1j * rng.standard_normal((n, 10)))
    dd = device_dictionary(atoms, dev)
    compare("cfg4-coh", torch.from_numpy(Z.astype(np.complex64)).to(dev), dd)
if "coh20" in which:
    cd, raw = workloads._offres_dictionary(1000, 20, 100, 100, 21, dev)
    atoms = cd.atoms_compressed
    del raw
    rng = np.random.default_rng(2)
    n = 65536
    idx = rng.integers(len(atoms), size=n)
    Z = atoms[idx] * rng.uniform(0.5, 1, size=(n, 1)) + 0.3 / np.sqrt(40) * (
        rng.standard_normal((n, 20)) + 1j * rng.standard_normal((n, 20)))
    dd = device_dictionary(atoms, dev)
    print("coh20 prefer_split", dd.prefer_split, "coherence", dd.bounds()["coherence"])
    compare("cfg2-coh", torch.from_numpy(Z.astype(np.complex64)).to(dev), dd)
