"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/s1/launches.csv [--skip N]

Prints, per kernel (template arguments kept), the launch count, total and mean
device time and the share of the summed device time.  ncu launch times are
cold-cache and serialised: compare shares, not absolutes.
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    n = 0
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        n += 1
        if n <= skip:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        ns = float(r[vi].replace(",", ""))
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ns)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'mean_us':>10s} {'share':>7s}")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:40s} {c:8d} {t / 1e3:10.1f} {t / c / 1e3:10.1f} {t / tot:7.3f}")
    print(f"{'TOTAL':40s} {sum(c for c, _ in agg.values()):8d} {tot / 1e3:10.1f}")


if __name__ == "__main__":
    main()
