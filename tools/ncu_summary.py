"""Markdown table from `ncu --page raw --csv` exports of single-kernel
captures (tools/final_round.sh): python tools/ncu_summary.py tag=file.csv[.gz] ..."""
import csv
import gzip
import sys

COLS = [("us", "gpu__time_duration.sum"),
        ("tensor_active_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        ("tensor_elapsed_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("xu_active_%", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        ("l2_%", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("dram_%", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("dram_read", "dram__bytes_read.sum"), ("dram_write", "dram__bytes_write.sum"),
        ("sm_clock", "smsp__cycles_elapsed.avg.per_second"),
        ("regs", "launch__registers_per_thread"), ("grid", "launch__grid_size"),
        ("issue_active_%", "smsp__issue_active.avg.pct_of_peak_sustained_active")]


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        rows = list(csv.reader(f))
    hdr, units = rows[0], rows[1]
    vals = rows[-1]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"


print("| kernel | " + " | ".join(c for c, _ in COLS) + " |")
print("|---|" + "---|" * len(COLS))
names = []
for arg in sys.argv[1:]:
    tag, path = arg.split("=", 1)
    d, name = load(path)
    names.append(f"{tag} = `{name[:60]}`")
    cells = []
    for _, m in COLS:
        v, u = d.get(m, ("", ""))
        cells.append(f"{v} {u}".strip())
    print(f"| {tag} | " + " | ".join(cells) + " |")
print()
print("Kernel names: " + "; ".join(names))
