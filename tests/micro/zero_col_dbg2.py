import sys, os, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "oracle"))
import oracle as orc, paper_1701_06600_b200 as pb
from test_gpu_lsq import collinear_factors, model_tensor, oracle_update
np.set_printoptions(precision=4, linewidth=200)
dims, r, s, seed = (48, 40, 36), 6, 120, 7
g = orc.Engine(4300 + seed, raw=True)
fs = collinear_factors(g, dims, r, 0.3, 2)
truth = [np.asfortranarray(g.matrix(dims[0], r)), np.asfortranarray(g.matrix(dims[1], r)), fs[2]]
x = model_tensor(np.ones(r), truth)
idx = orc.sample_tables(dims, s, seed, 1)[0][0]
xh = orc.mix_tensor(x, "dct", seed)
for tr in (None, "dct"):
    got, glam, rank = pb.mode_update(xh if tr else x, 0, idx, fs, np.ones(r), True, tr, seed) if tr else pb.mode_update(x, 0, idx, fs, np.ones(r), True)
    want, wlam, zs = oracle_update(orc, x, 0, idx, fs, np.ones(r), True, mix=tr, seed=seed)
    print(tr, "rank", rank, "col diffs", np.linalg.norm(got - want, axis=0), "glam", glam, "wlam", wlam)
    print(" gpu col2", got[:4, 2], "orc", want[:4, 2])
