"""Compact view of an ncu report: details page (section / metric / value) and
the top source lines by warp stall samples.  usage: ncu_details.py rep [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name"):
        print(f"{d['Section Name'][:28]:28s} {d['Metric Name'][:44]:44s} {d['Metric Value']:>14s} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if rows and rows[0] and rows[0][0] == "Kernel Name":
    rows = rows[1:]
if rows:
    h = rows[0]
    key = next((k for k in h if "Warp Stall Sampling (All" in k), None)
    if key:
        items = []
        for r in rows[1:]:
            d = dict(zip(h, r))
            try:
                items.append((float(d[key] or 0), d.get("Source", "")[:110], d.get("Address", "")))
            except ValueError:
                pass
        tot = sum(i[0] for i in items) or 1
        print("\nTop SASS by stall samples:")
        for v, s, a in sorted(items, reverse=True)[:25]:
            print(f"{100 * v / tot:5.1f}%  {a}  {s}")
