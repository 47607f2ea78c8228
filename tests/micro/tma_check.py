"""Debug: TMA mixing pass (v3) vs v2 vs the oracle, per shape (not part of the product)."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as orc  # noqa: E402
import paper_1701_06600_b200 as pb  # noqa: E402

for dims in [(200, 120, 64), (200, 8, 8), (16, 120, 8), (16, 8, 64), (64, 40, 48, 32)]:
    x = orc.random_tensor(dims, 5)
    t = pb.DeviceTensor(dims)
    t.upload(x)
    t.mix("dct", 3)
    v3 = t.download()
    t.upload(x)
    os.environ["CPRAND_MIX_V2"] = "1"
    t.mix("dct", 3)
    del os.environ["CPRAND_MIX_V2"]
    v2 = t.download()
    t.close()
    want = orc.mix_tensor(x, "dct", 3)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    print(dims, "v3-v2 bitwise", np.array_equal(v3, v2), "rel v3", rel(v3, want), "rel v2", rel(v2, want),
          "max|v3-v2|", float(np.max(np.abs(v3 - v2))), flush=True)
