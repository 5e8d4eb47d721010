"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list:
per-kernel launches, ms per apply and share.   python tools/launch_summary.py X [n_applies]"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    for r in rows[1:]:
        name = re.sub(r"^qbxg::(<unnamed>::)?", "", re.sub(r"\(.*", "", r[ki]))
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot / reps:.2f} ms per apply over {reps} applies (setup kernels included)")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:48]:48s} {n:6d} {t / reps:9.3f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main()
