"""Executor trace of a bench workload (default GPT-1.3B, vertical, alpha 0.2,
split (1,1,1)), middle of the iterations: per-phase resource busy time,
compute-stream gaps attributed to the plan dependency that finished last
before each compute task started, and per-stage timing.

usage: python tools/trace_phase.py [M] [opt_tier] [host_threads] [--config NAME] [--ring R]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("M", nargs="?", type=int, default=0)
ap.add_argument("tier", nargs="?", type=int, default=-1)
ap.add_argument("threads", nargs="?", type=int, default=0)
ap.add_argument("--config", default="gpt1.3b")
ap.add_argument("--ring", type=int, default=0, help="ssd_ring_layers override")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
N, h, H, s, b, V, M, split, alpha, tier, ring = CONFIGS[a.config]
M = a.M or M
tier = tier if a.tier < 0 else a.tier
ring = a.ring or ring
threads = a.threads
model = gs.ModelSpec(N, h, H, s, b, 2, 4, 3, 1)
plan = gs.build_vertical(model, M, gs.StorageSplit(*split), alpha)
eng = gs.Engine(plan, model, V, gs.AdamConfig(1e-4), opt_tier=tier, record_trace=True,
                host_threads=threads, ssd_ring_layers=ring, nvme_dir=os.environ.get("GS_NVME_DIR", "/tmp"))
tok = np.random.default_rng(7).integers(0, V, size=(a.iters, M, b, s + 1), dtype=np.int32)
eng.run(tok[:1])
rep = eng.run(tok)
print(f"{a.config} M={M} opt_tier={tier} ring={ring} host_threads={threads}: total ms {rep.total_ms:.1f}, "
      f"per iteration {rep.total_ms / a.iters:.1f}")
tasks = [plan.task(i) for i in range(len(plan))]
recs = {r["task"]: r for r in rep.trace if r["iteration"] == 1}
prev = {r["task"]: r for r in rep.trace if r["iteration"] == 0}
t0 = min(r["t_start_ms"] for r in recs.values())
t1 = max(r["t_end_ms"] for r in recs.values())
print(f"iteration 1 span {t1 - t0:.1f} ms")
gpu = sorted([r for r in recs.values() if r["resource"] == "compute"], key=lambda r: r["t_start_ms"])
first_bwd = min(r["t_start_ms"] for r in gpu if tasks[r["task"]]["kind"] == "bwd")


def union(iv):
    iv = sorted(iv)
    tot, cur_s, cur_e = 0.0, None, None
    for a, e in iv:
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = a, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


for phase, lo, hi in (("fwd", t0, first_bwd), ("bwd", first_bwd, t1)):
    print(f"--- {phase} phase {hi - lo:.1f} ms")
    for res in gs.RESOURCES:
        iv = [(max(lo, r["t_start_ms"]), min(hi, r["t_end_ms"])) for r in recs.values()
              if r["resource"] == res and r["t_end_ms"] > lo and r["t_start_ms"] < hi]
        byts = sum(r["bytes"] for r in recs.values() if r["resource"] == res and lo <= r["t_start_ms"] < hi)
        print(f"  {res:9s} busy(union) {union(iv):8.1f} ms  bytes {byts / 1e9:7.2f} GB")
# gaps attributed to the last-finishing plan dependency
attr = {}
gaps = []
for a, c in zip(gpu, gpu[1:]):
    gap = c["t_start_ms"] - a["t_end_ms"]
    if gap <= 0.005:
        continue
    t = tasks[c["task"]]
    best, best_end = None, -1e9
    for dep in t["deps"]:
        r = recs.get(dep)
        if r and r["t_end_ms"] > best_end:
            best, best_end = dep, r["t_end_ms"]
    cd = t.get("cross_iter_dep", -1)
    if cd is not None and cd >= 0 and cd in prev and prev[cd]["t_end_ms"] > best_end:
        best, best_end = cd, prev[cd]["t_end_ms"]
    if best is None or best_end < a["t_end_ms"] - 0.005:
        key = "none (host dispatch / hazard edge)"
    else:
        d = tasks[best]
        key = f"{d['kind']}:{d.get('data', '')}:{d.get('link', '')}"
    attr[key] = attr.get(key, 0.0) + gap
    gaps.append((gap, a["task"], c["task"], key))
print("compute gaps total ms", round(sum(g[0] for g in gaps), 2))
for k, v in sorted(attr.items(), key=lambda kv: -kv[1]):
    print(f"  waiting on {k:40s} {v:8.2f} ms")
gaps.sort(reverse=True)
for gap, a, c, key in gaps[:12]:
    ta, tc = tasks[a], tasks[c]
    print(f"  gap {gap:6.2f} ms {ta['kind']} L{ta['layer']} mb{ta['microbatch']} st{ta['stage']} -> "
          f"{tc['kind']} L{tc['layer']} mb{tc['microbatch']} st{tc['stage']}  [{key}]")
for kind in ("fwd", "bwd", "fixed_ops"):
    dd = [r["t_end_ms"] - r["t_start_ms"] for r in gpu if tasks[r["task"]]["kind"] == kind]
    if dd:
        print(f"{kind:9s} n {len(dd):4d} mean {np.mean(dd):.3f} ms sum {np.sum(dd):.1f}")
cpu = sorted([r for r in recs.values() if r["resource"] == "cpu_step"], key=lambda r: r["t_start_ms"])
for r in cpu[:3] + cpu[-3:]:
    t = tasks[r["task"]]
    print(f"cpu_step L{t['layer']} st{t['stage']} elems {t.get('elements')} {r['t_end_ms'] - r['t_start_ms']:.2f} ms "
          f"-> {t.get('elements', 0) / max(1e-9, (r['t_end_ms'] - r['t_start_ms']) / 1e3) / 1e9:.2f} Gelem/s")

# window around the worst backward gaps: every transfer / step task that
# overlaps it, with its times relative to the gap start
for gap, a, c, key in ([g for g in gaps if tasks[g[2]]["kind"] != "bwd"][:1] +
                       [g for g in gaps if tasks[g[2]]["kind"] == "bwd"][:2]):
    ga, gc = recs[a]["t_end_ms"], recs[c]["t_start_ms"]
    print(f"=== window: gap {gap:.2f} ms before {tasks[c]['kind']} L{tasks[c]['layer']} mb{tasks[c]['microbatch']} st{tasks[c]['stage']}")
    win = [r for r in recs.values() if r["t_end_ms"] > ga - (25 if r["resource"] != "compute" else 4)
           and r["t_start_ms"] < gc + 1]
    for r in sorted(win, key=lambda r: (r["resource"], r["t_start_ms"])):
        t = tasks[r["task"]]
        print(f"  {r['resource']:9s} id {r['task']:5d} {t['kind']:8s} {t.get('data', ''):15s} L{t['layer']:<3d} "
              f"mb{t['microbatch']:<3d} st{t['stage']:<3d} {r['t_start_ms'] - ga:8.2f} .. {r['t_end_ms'] - ga:8.2f} ms "
              f"{t.get('bytes', 0) / 1e6:8.1f} MB host {r['t_host_ms'] - ga:8.2f} deps {t['deps']}")

# NVMe queues: per-task bandwidth and the idle gaps between consecutive tasks
for res in ("ssd_read", "ssd_write"):
    rs = sorted([r for r in recs.values() if r["resource"] == res], key=lambda r: r["t_start_ms"])
    if not rs:
        continue
    busy = sum(r["t_end_ms"] - r["t_start_ms"] for r in rs)
    byts = sum(r["bytes"] for r in rs)
    gaps = [b["t_start_ms"] - a["t_end_ms"] for a, b in zip(rs, rs[1:])]
    print(f"{res}: {len(rs)} tasks, {byts / 1e9:.2f} GB, busy {busy:.0f} ms -> {byts / 1e6 / max(busy, 1e-9):.2f} GB/s "
          f"while busy; gaps between tasks: total {sum(g for g in gaps if g > 0):.0f} ms, "
          f"max {max(gaps) if gaps else 0:.0f} ms")
    sizes = sorted({round(r['bytes'] / 1e6) for r in rs})
    for mb in sizes:
        sel = [r for r in rs if round(r["bytes"] / 1e6) == mb]
        d = [r["t_end_ms"] - r["t_start_ms"] for r in sel]
        print(f"   {mb:8d} MB x {len(sel):3d}: mean {np.mean(d):8.1f} ms -> {mb / np.mean(d):.2f} GB/s")
    if os.environ.get("GS_TRACE_SSD_LIST"):
        for r in rs:
            t = tasks[r["task"]]
            print(f"     {res} id {r['task']:6d} {t.get('data', ''):10s} L{t['layer']:<3d} st{t['stage']:<4d} "
                  f"{r['t_start_ms'] - t0:9.1f} .. {r['t_end_ms'] - t0:9.1f} ms  {r['bytes'] / 1e6:8.1f} MB "
                  f"host {r['t_host_ms'] - t0:9.1f}")
