"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name, launch count, mean duration and share of the listed time.

    python tools/launch_summary.py launches.csv "header line" > profiles/<round>_launches_<cfg>_summary.txt

ncu serialises launches and runs them cold-cache, so compare shares, not
absolute times, with bench.py's CUDA-event numbers.
"""
import csv
import sys
from collections import OrderedDict


def main(path, header=""):
    rows = list(csv.reader(open(path)))
    try:
        h = next(r for r in rows if "Kernel Name" in r)
    except StopIteration:
        print("no launches in", path)
        return
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    agg = OrderedDict()
    for r in rows[rows.index(h) + 1:]:
        if len(r) != len(h) or r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:60]
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ms)
    total = sum(t for _, t in agg.values())
    if header:
        print(header)
    print("cold-cache, serialised per-launch times; compare shares")
    for name, (c, t) in agg.items():
        print(f"{name:60s} launches {c:3d}  mean {t / c:9.3f} ms  share {100 * t / total:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:3])
