"""Development aid: run the tcgen05 projection for one (n, d) and compare with the FFMA path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_01967_b200 as cb
n, d = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(0)
a = rng.standard_normal((d, 10)) + 1j * rng.standard_normal((d, 10))
a /= np.linalg.norm(a, axis=1)[:, None]
Z = rng.standard_normal((n, 10)) + 1j * rng.standard_normal((n, 10))
r1 = cb.project_cone_exact(Z, a, algo="tcgen05")
torch.cuda.synchronize()
r2 = cb.project_cone_exact(Z, a, algo="ffma")
print(n, d, "mismatch", int((r1.indices != r2.indices).sum()), flush=True)
