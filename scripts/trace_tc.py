"""Per-hop latency trace of the tcgen05 pipeline (development aid; needs the TRACE=1 build)."""
import ctypes, os, sys
os.environ.setdefault("CBB_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1810_01967_b200", "libcoverblip_b200_trace.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_01967_b200 as cb
from paper_1810_01967_b200 import _lib
from paper_1810_01967_b200.workloads import random_atoms, cone_voxels
from paper_1810_01967_b200.projection import project_device
N = 1 << 18; D = 1 << 17
atoms = random_atoms(D, 10, seed=0)
Z, _ = cone_voxels(atoms, N, seed=1, dtype=np.complex64)
dd = cb.device_dictionary(atoms); zt = torch.from_numpy(Z).cuda()
for _ in range(3):
    project_device(zt, dd, algo=os.environ.get("TRACE_ALGO", "tcgen05"), proj_c128=False)
torch.cuda.synchronize()
lib = _lib.load()
fn = lib.cbb_dev_trace_dump; fn.restype = ctypes.c_int; fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
T = 2048
buf = np.zeros(T * 8, dtype=np.int64)
assert fn(buf.ctypes.data, T) == 0
t = buf.reshape(T, 8).astype(np.float64)
ks = np.arange(200, 1900)
def med(x): return float(np.median(x))
print("issuer: data wait after acc_free (4->0)", med(t[ks, 0] - t[ks, 4]))
print("release(k-3) -> acc_free seen (3->4)", med(t[ks, 4] - t[ks - 3, 3]))
print("issuer: issue+commit (0->1)         ", med(t[ks, 1] - t[ks, 0]))
print("issuer: loop overhead (1 -> next 4) ", med(t[ks + 3, 4] - t[ks, 1]))
print("epi: wait t_full (5->2)             ", med(t[ks, 2] - t[ks, 5]))
print("epi: load (2->3)                    ", med(t[ks, 3] - t[ks, 2]))
print("epi: screen (3->6)                  ", med(t[ks, 6] - t[ks, 3]))
print("epi: loop overhead (6 -> next 5)    ", med(t[ks + 3, 5] - t[ks, 6]))
print("epi: part period (2 -> next 2)      ", med(t[ks + 3, 2] - t[ks, 2]))
print("commit -> t_full ready (1->2)       ", med(t[ks, 2] - t[ks, 1]))
print("release(k-3) -> issuer ready (3->0) ", med(t[ks, 0] - t[ks - 3, 3]))
print("producer issue(k) -> issuer ready   ", med(t[ks, 0] - t[ks, 7]))
KS = int(os.environ.get("TRACE_STAGES", "9"))
print("commit(k) -> producer issue(k+S)    ", med(t[ks + KS, 7] - t[ks, 1]), "(S = %d)" % KS)
print("tile period (issuer ready k -> k+1) ", med(t[ks + 1, 0] - t[ks, 0]))
print("frac of part time waiting           ", med((t[ks, 2] - t[ks, 5]) / (t[ks + 3, 2] - t[ks, 2])))
vt = np.zeros(256 * 4, dtype=np.int64)
assert fn(vt.ctypes.data, -1) == 0
vt = vt.reshape(256, 4).astype(np.float64)
nv = int((vt[:, 0] > 0).sum())
its = np.arange(1, nv - 1)
print("voxel tiles traced                  ", nv)
print("voxel tile: atom loop (0->1)        ", med(vt[its, 1] - vt[its, 0]))
print("voxel tile: finalize (1->2)         ", med(vt[its, 2] - vt[its, 1]))
print("voxel tile: total (0 -> next 0)     ", med(vt[its + 1, 0] - vt[its, 0]))
print("voxel tile 0: loop / finalize       ", vt[0, 1] - vt[0, 0], vt[0, 2] - vt[0, 1])
