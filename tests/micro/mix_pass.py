"""Run the whole-tensor mixing pass once per mode on a 1000^3 tensor (for ncu)."""
import sys
sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
import paper_1701_06600_b200 as pb
dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (1000, 1000, 1000)
t = pb.DeviceTensor(dims)
t.synth(5, 0.0, 0.0, 1)
print("ms per mode", t.mix("dct", 1), flush=True)
print("ms per mode", t.mix("dct", 1), flush=True)
