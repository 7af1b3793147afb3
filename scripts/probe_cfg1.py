"""Quick timing probe of the cfg1 projection (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_01967_b200 as cb
from paper_1810_01967_b200.workloads import random_atoms, cone_voxels
from paper_1810_01967_b200.projection import project_device, overflow_count

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
D = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 17
algos = sys.argv[3].split(",") if len(sys.argv) > 3 else ["tcgen05"]
t0 = time.time()
atoms = random_atoms(D, 10, seed=0)
Z, gen = cone_voxels(atoms, N, seed=1, dtype=np.complex64)
print(f"gen {time.time()-t0:.1f}s", flush=True)
dd = cb.device_dictionary(atoms)
zt = torch.from_numpy(Z).cuda()
for algo in algos:
    for it in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        idx, gam, proj = project_device(zt, dd, algo=algo, proj_c128=False)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        flops = 4 * 10 * N * D
        print(f"{algo} it{it}: {ms:.3f} ms  {flops/ms/1e9:.1f} TFLOP/s algorithmic  overflow={overflow_count(N,10)}", flush=True)
    agree = (idx.cpu().numpy() == gen).mean()
    print(f"{algo}: argmax==generator {agree:.4f}")
