"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total and mean duration, share of the listed time.

    python tools/ncu_launch_summary.py gpurun_out/launches.csv [--skip REGEX]
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    skip = re.compile(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else None
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    unit = ""
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        unit = r[ui]
        n, t = agg.get(r[ki], (0, 0.0))
        agg[r[ki]] = (n + 1, t + v)
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    total = sum(t for k, (n, t) in agg.items() if not (skip and skip.search(k)))
    print(f"# {path}: {sum(n for n, _ in agg.values())} launches (gpu__time_duration.sum, cold-cache, serialised)")
    print(f"{'launches':>8} {'total ms':>10} {'mean ms':>9} {'share':>6}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = "" if skip and skip.search(k) else f"{100 * t / total:5.1f}%"
        print(f"{n:8d} {t * scale:10.3f} {t * scale / n:9.4f} {share:>6}  {k[:110]}")
    if skip:
        print(f"# share excludes kernels matching {skip.pattern!r} (store upload / probes outside the timed step)")


if __name__ == "__main__":
    main()
