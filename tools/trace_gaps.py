"""Per-resource busy time and the largest compute-stream gaps of one
iteration of the GPT-1.3B bench workload (executor trace, CUDA events)."""
import json
import sys

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_bindings as ob  # noqa: E402
import paper_2512_17570_b200 as gs  # noqa: E402

N, h, H, s, b, V, M = 24, 2048, 16, 2048, 2, 50304, int(sys.argv[1]) if len(sys.argv) > 1 else 16
alpha = 0.2
model = gs.ModelSpec(N, h, H, s, b, 2, 4, 3, 1)
plan = gs.build_vertical(model, M, gs.StorageSplit(1, 1, 1), alpha)
eng = gs.Engine(plan, model, V, gs.AdamConfig(1e-4), record_trace=True)
g = ob.Geometry(n_layers=N, hidden=h, heads=H, seq=s, mb_size=b, vocab=V)
tok = ob.make_tokens(g, 3, M)
rep = eng.run(tok)
print("total ms", rep.total_ms, "per iteration", rep.total_ms / 3)
tasks = [plan.task(i) for i in range(len(plan))]
it = 1
recs = [r for r in rep.trace if r["iteration"] == it]
t0 = min(r["t_start_ms"] for r in recs); t1 = max(r["t_end_ms"] for r in recs)
print("iteration", it, "span ms", t1 - t0)
for res in gs.RESOURCES:
    rr = sorted([r for r in recs if r["resource"] == res], key=lambda r: r["t_start_ms"])
    if not rr:
        continue
    busy = sum(r["t_end_ms"] - r["t_start_ms"] for r in rr)
    print(f"{res:10s} tasks {len(rr):5d} busy {busy:9.1f} ms  first {rr[0]['t_start_ms']-t0:8.1f} last {rr[-1]['t_end_ms']-t0:8.1f}")
gpu = sorted([r for r in recs if r["resource"] == "compute"], key=lambda r: r["t_start_ms"])
gaps = []
for a, c in zip(gpu, gpu[1:]):
    gaps.append((c["t_start_ms"] - a["t_end_ms"], a["task"], c["task"]))
gaps.sort(reverse=True)
print("compute gaps total ms", sum(g_[0] for g_ in gaps))
for gap, a, c in gaps[:15]:
    ta, tc = tasks[a], tasks[c]
    print(f"gap {gap:7.2f} ms after {ta['kind']} L{ta['layer']} mb{ta['microbatch']} st{ta['stage']} -> {tc['kind']} L{tc['layer']} mb{tc['microbatch']} st{tc['stage']}")
# task durations by kind
for kind in ("fwd", "bwd", "fixed_ops"):
    d = [r["t_end_ms"] - r["t_start_ms"] for r in gpu if tasks[r["task"]]["kind"] == kind]
    if d:
        print(kind, "n", len(d), "mean ms", np.mean(d), "max", np.max(d), "sum", np.sum(d))
cpu = [r for r in recs if r["resource"] == "cpu_step"]
print("cpu_step sum ms", sum(r["t_end_ms"] - r["t_start_ms"] for r in cpu))
# PCIe copy behaviour: per-task achieved rate and the idle time between
# consecutive copies on each copy stream, forward vs backward phase
first_bwd = min(r["t_start_ms"] for r in gpu if tasks[r["task"]]["kind"] == "bwd")
for res in ("pcie_h2d", "pcie_d2h"):
    rr = sorted([r for r in recs if r["resource"] == res], key=lambda r: r["t_start_ms"])
    for phase, sel in (("fwd", lambda r: r["t_end_ms"] <= first_bwd), ("bwd", lambda r: r["t_start_ms"] >= first_bwd)):
        ph = [r for r in rr if sel(r)]
        if not ph:
            continue
        rates = [r["bytes"] / max(1e-9, (r["t_end_ms"] - r["t_start_ms"]) / 1e3) / 1e9 for r in ph if r["bytes"] > (4 << 20)]
        idle = sum(max(0.0, b["t_start_ms"] - a["t_end_ms"]) for a, b in zip(ph, ph[1:]))
        span = ph[-1]["t_end_ms"] - ph[0]["t_start_ms"]
        byts = sum(r["bytes"] for r in ph)
        print(f"{res} {phase}: {len(ph)} copies, {byts / 1e9:.2f} GB in {span:.1f} ms span "
              f"({byts / 1e9 / (span / 1e3):.1f} GB/s), idle between copies {idle:.1f} ms, "
              f"median copy rate {np.median(rates) if rates else 0:.1f} GB/s")

# One forward stage in detail: every task on every resource, times relative to
# the stage's first compute task.
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 6
st_tasks = [r for r in gpu if tasks[r["task"]]["kind"] == "fwd" and tasks[r["task"]]["stage"] == stage]
ts0 = min(r["t_start_ms"] for r in st_tasks); ts1 = max(r["t_end_ms"] for r in st_tasks)
print(f"\nforward stage {stage}: compute {ts0 - t0:.2f} .. {ts1 - t0:.2f} ms ({ts1 - ts0:.2f} ms, {len(st_tasks)} tasks)")
window = [r for r in recs if r["t_end_ms"] >= ts0 - 2 and r["t_start_ms"] <= ts1 + 2]
d2h = [r for r in recs if r["resource"] == "pcie_d2h"]
for r in sorted(window, key=lambda r: (r["resource"], r["t_start_ms"])):
    t = tasks[r["task"]]
    dur = r["t_end_ms"] - r["t_start_ms"]
    ov = 0.0
    if r["resource"] == "pcie_h2d":
        for q in d2h:
            ov += max(0.0, min(q["t_end_ms"], r["t_end_ms"]) - max(q["t_start_ms"], r["t_start_ms"]))
    rate = r["bytes"] / max(1e-9, dur / 1e3) / 1e9 if r["bytes"] else 0.0
    print(f"  {r['resource']:9s} {t['kind']:12s} L{t['layer']:<3d} mb{t['microbatch']:<3d} "
          f"{r['t_start_ms'] - ts0:8.3f} {r['t_end_ms'] - ts0:8.3f}  {r['bytes'] / 1e6:8.2f} MB  {rate:6.1f} GB/s"
          + (f"  d2h-overlap {ov / max(dur, 1e-9):.2f}" if r["resource"] == "pcie_h2d" else ""))
