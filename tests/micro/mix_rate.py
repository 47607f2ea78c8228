"""Whole-tensor mixing pass: TB/s per mode (16 B / element) for the current
kernel selection vs the v2 / v3 kernels (env switches), on C5 (320^4) and
C3-like shapes, plus an accuracy check of fibers against the oracle."""
import os
import subprocess
import sys
ROOT = __file__.rsplit("/tests/", 1)[0]
sys.path.insert(0, ROOT)
sys.path.insert(0, ROOT + "/oracle")
import numpy as np  # noqa: E402
import paper_1701_06600_b200 as pb  # noqa: E402

dims = tuple(int(a) for a in sys.argv[1].split(",")) if len(sys.argv) > 1 else (320, 320, 320, 320)
p = int(np.prod(dims))
t = pb.DeviceTensor(dims)
t.synth(5, 0.0, 0.01, 1)
t.mix("dct", 1)  # warm
ms = t.mix("dct", 1)
print(dims, os.environ.get("CPRAND_MIX_V2", ""), os.environ.get("CPRAND_MIX_TMA", ""),
      "TB/s per mode", [round(16 * p / (m * 1e-3) / 1e12, 2) for m in ms], flush=True)
if len(sys.argv) > 2:  # accuracy vs the oracle on random fibers, mode by mode
    import oracle as orc
    t.synth(5, 0.0, 0.01, 1)
    signs = orc.mixing_signs(dims, "dct", 1)
    g = orc.Engine(5, raw=True)
    for m in range(len(dims)):
        idx = orc.draw_samples(g, dims, m, 200)
        before = t.read_fibers(m, idx)
        t.mix_modes("dct", 1, m, m + 1)
        after = t.read_fibers(m, idx)
        want = np.stack([orc.transform("dct", signs[m] * before[:, j]) for j in range(idx.shape[0])], axis=1)
        print("mode", m, "max rel err", max(np.linalg.norm(after[:, j] - want[:, j]) / np.linalg.norm(want[:, j])
                                             for j in range(idx.shape[0])), flush=True)
