"""Hot SASS lines (warp-stall samples) of an ncu report, with context (dev helper)."""
import csv
import io
import subprocess
import sys

path, ntop = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for r in csv.reader(io.StringIO(out)):
    if len(r) > 14 and r[-3] in ("Duration", "Elapsed Cycles", "Grid Size", "Block Size"):
        print(r[-3], r[-1], r[-2])
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(int(d[key] or 0) for d in data)
print("total samples", tot)
top = sorted(range(len(data)), key=lambda i: -int(data[i][key] or 0))[:ntop]
for i in sorted(top):
    print("----")
    for k in range(max(0, i - 4), i + 1):
        d = data[k]
        print(d[key].rjust(5), d["Address"][-5:], d["Source"][:90])
