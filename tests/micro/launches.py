"""Summarise an ncu --csv launch list: per-kernel count, mean time, mean DRAM read."""
import csv
import sys
from collections import defaultdict

UNIT = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}


def main(path, skip_prefix=("synth",)):
    rows = list(csv.reader(open(path)))
    hdr, per = None, defaultdict(dict)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            per[(int(d["ID"]), d["Kernel Name"])][d["Metric Name"]] = (
                float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for (i, n), m in per.items():
        short = n.split("(")[0].replace("void ", "").split("::")[-1]
        if short.startswith(skip_prefix):
            continue
        t = m["gpu__time_duration.sum"]
        b = m.get("dram__bytes_read.sum", (0.0, "byte"))
        a = agg[short]
        a[0] += 1
        a[1] += t[0] * (1e-3 if t[1] == "ns" else 1.0)
        a[2] += b[0] * UNIT.get(b[1], 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':40s} {'n':>4s} {'us/launch':>10s} {'MB/launch':>10s} {'share':>6s}")
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:40s} {c:4d} {t / c:10.2f} {b / c:10.2f} {t / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
