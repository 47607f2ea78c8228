"""Aggregate ncu source-page CSV (--print-source cuda,sass) per CUDA source line.
usage: python srcprof.py report.ncu-rep [top]"""
import csv, subprocess, sys, collections

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
agg = collections.Counter()
stall = collections.defaultdict(collections.Counter)
text = {}
fname = None
hdr = None
cur = None
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] == "Function Name":
        continue
    if row[0]:
        cur = (fname, int(row[0]))
        text[cur] = row[1][:90]
    try:
        v = float(row[4])
    except (ValueError, IndexError):
        continue
    agg[cur] += v
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stall[cur][h[6:]] += float(row[i])
            except ValueError:
                pass
tot = sum(agg.values()) or 1
print(f"total samples {tot:.0f}")
for k, v in agg.most_common(top):
    st = ",".join(f"{a}:{b/v*100:.0f}" for a, b in stall[k].most_common(3))
    print(f"{v/tot*100:5.1f}% {k[0]}:{k[1]:<4} {text.get(k,'')}   [{st}]")
