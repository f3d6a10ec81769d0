"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum launch list
(CSV from tools/launch_list*.sh): launches, share, average duration."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        out.append((r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", ""), v))
    return out


def main(path):
    ks = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us in ks:
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{len(ks)} launches, kernel time {tot / 1e3:.1f} ms")
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name[:64]:64s} {n:6d} {100 * t / tot:6.2f}%  avg {t / n:9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
