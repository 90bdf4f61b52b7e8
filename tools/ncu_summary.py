"""Summarise ncu reports into profiles/ (text + JSON), run here (no GPU needed).

usage: python tools/ncu_summary.py <tag> <report.ncu-rep> [<report> ...]
       python tools/ncu_summary.py --launches <launches.csv> <out.txt>
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic"]
UNIT = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def to_bytes(v, u):
    return float(v.replace(",", "")) * UNIT.get(u, 1.0)


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    tot, lines = {}, []
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0]
        ns = float(d["Metric Value"].replace(",", ""))
        ns *= {"usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9}.get(d["Metric Unit"], 1.0)
        tot[name] = tot.get(name, 0.0) + ns
        lines.append(f"{name:60s} {ns / 1e3:10.2f} us")
    s = sum(tot.values())
    lines.append("\nshare of device time (cold-cache, serialised launches):")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"  {k:58s} {100 * v / s:6.2f} %")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def main():
    if sys.argv[1] == "--launches":
        return launches(sys.argv[2], sys.argv[3])
    tag = sys.argv[1]
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for path in sys.argv[2:]:
        name = os.path.basename(path).replace(".ncu-rep", "")
        txt = []
        for d, u in raw(path):
            txt.append(f"## {d.get('Kernel Name', '?')}")
            for k in KEYS:
                if k in d:
                    txt.append(f"{k:62s} {d[k]} {u[k]}")
            rb = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
            wb = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
            dur = float(d["gpu__time_duration.sum"].replace(",", ""))
            dur *= {"usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6, "second": 1e3, "s": 1e3}.get(u["gpu__time_duration.sum"], 1.0)
            rec = {"kernel": d.get("Kernel Name", "?")[:90], "duration_ms": dur, "dram_bytes_per_launch": rb + wb,
                   "capture": f"{tag}:{name}"}
            summ[f"{tag}:{name}"] = rec
            summ[f"latest:{name}"] = rec  # what bench.py reads
        out = os.path.join(ROOT, "profiles", f"{tag}_{name}.txt")
        open(out, "w").write("\n".join(txt) + "\n")
        print(open(out).read())
    json.dump(summ, open(summ_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
