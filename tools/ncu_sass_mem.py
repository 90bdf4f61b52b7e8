"""Per-SASS-instruction memory attribution of an ncu report's source page (dev helper):
shared wavefronts, global tag requests, L2 sectors, stall samples of the heavy instructions."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.003
if path.endswith(".csv"):
    out = open(path).read()
else:
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


cols = ["Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "L1 Tag Requests Global",
        "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Ideal", "Warp Stall Sampling (All Samples)"]
tot = {c: sum(I(d[c]) for d in data) for c in cols}
print({c: tot[c] for c in cols})
print("addr inst shWf shIdeal tags sectors secIdeal samples source")
for d in data:
    if any(I(d[c]) > tot[c] * frac for c in ("L1 Wavefronts Shared", "L1 Tag Requests Global",
                                              "L2 Theoretical Sectors Global", "Warp Stall Sampling (All Samples)")):
        print(d["Address"][-5:], *[I(d[c]) for c in cols], d["Source"][:60])
