import sys, os
sys.path.insert(0, "/root/repo")
import paper_1701_06600_b200 as pb
for dims in [(1000, 1000, 1000), (80, 80, 80, 80), (320, 320, 320, 40)]:
    t = pb.DeviceTensor(dims)
    t.synth(5, 0.0, 0.0, 1)
    t.mix("dct", 1)
    ms = t.mix("dct", 1)
    p = 1
    for d in dims: p *= d
    print(dims, "v3 ms", [round(m, 3) for m in ms], "TB/s", [round(16 * p / (m * 1e-3) / 1e12, 2) for m in ms], flush=True)
    os.environ["CPRAND_MIX_V2"] = "1"
    ms = t.mix("dct", 1)
    del os.environ["CPRAND_MIX_V2"]
    print(dims, "v2 ms", [round(m, 3) for m in ms], "TB/s", [round(16 * p / (m * 1e-3) / 1e12, 2) for m in ms], flush=True)
    t.close()
