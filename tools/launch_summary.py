"""Per-kernel summary of an ncu launch list (CSV from tools/launch_list*.sh):
launches, share of device time, average duration and — when the list holds
dram__bytes_read/write.sum — average DRAM bytes per launch.
Usage: python tools/launch_summary.py launches.csv [--json out.json]"""
import collections
import gzip
import csv
import json
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ii, ki = hdr.index("ID"), hdr.index("Kernel Name")
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    launches = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        k = launches.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            k["us"] = v * SCALE.get(r[ui], 1.0)
        elif r[mi].startswith("dram__bytes"):
            k["dram"] = k.get("dram", 0.0) + v * BYTES.get(r[ui], 1.0)
    return list(launches.values())


def summarize(ks):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k in ks:
        a = agg[k["name"]]
        a[0] += 1
        a[1] += k.get("us", 0.0)
        a[2] += k.get("dram", 0.0)
    return agg


def main(path, out_json=None):
    ks = load(path)
    agg = summarize(ks)
    tot = sum(v[1] for v in agg.values())
    print(f"{len(ks)} launches, kernel time {tot / 1e3:.1f} ms")
    for name, (n, t, d) in sorted(agg.items(), key=lambda x: -x[1][1]):
        extra = f"  dram {d / n / 1e6:8.1f} MB/launch" if d else ""
        print(f"{name[:64]:64s} {n:6d} {100 * t / tot:6.2f}%  avg {t / n:9.1f} us{extra}")
    gemm = [k for k in ks if "tc_gemm_kernel" in k["name"]]
    if out_json and gemm:
        res = {"source": path, "launches": len(ks), "kernel_ms": tot / 1e3,
               "gemm_launches": len(gemm), "gemm_share": sum(k.get("us", 0) for k in gemm) / tot,
               "gemm_dram_bytes_per_launch": sum(k.get("dram", 0.0) for k in gemm) / len(gemm),
               "gemm_us_per_launch": sum(k.get("us", 0.0) for k in gemm) / len(gemm)}
        json.dump(res, open(out_json, "w"), indent=1)
        print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--json" else None)
