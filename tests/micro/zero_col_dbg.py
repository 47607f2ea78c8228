import sys, os, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "oracle"))
import oracle as orc, paper_1701_06600_b200 as pb
from test_gpu_lsq import session_first_mode
np.set_printoptions(precision=4, linewidth=200)
cols = {}
for method, fused, tr in [("rand", 0, None), ("mix", -1, "dct"), ("mix", 0, "dct")]:
    res, out, lam = session_first_mode(pb, orc, method, fused, 0.3, zero_col=2, transform=tr)
    got, want, zs = out[0]
    cols[(method, fused)] = (got[:, 2].copy(), want[:, 2].copy())
    print(method, fused, "gpu col2[:6]", got[:6, 2], "norm", np.linalg.norm(got[:, 2]))
    print(method, fused, "orc col2[:6]", want[:6, 2], "norm", np.linalg.norm(want[:, 2]))
    print("zs col2 norm", np.linalg.norm(zs[:, 2]), "lam", res.lam)
np.savez(os.path.join(os.path.dirname(__file__), "..", "..", "gpurun_out", "zc.npz"),
         rand=cols[("rand", 0)][0], mixf=cols[("mix", -1)][0], mixc=cols[("mix", 0)][0], orc=cols[("rand", 0)][1])
