"""bench.py — throughput of the GreedySnake hot path on B200.

A step is one training iteration of the vertical (snake) plan with the
alpha-delayed optimizer step, executed by the B200 executor through the
C-ABI (gs_engine_run): every plan task runs for real (tcgen05 GEMMs, flash
attention, fused Adam, PCIe DMA of params / checkpoints / gradients /
optimizer state, NVMe I/O when the split puts data on SSD).

Workload (BASELINE.json configs[1], as written): GPT-1.3B (N=24, h=2048, 16
heads, s=2048, b=2, vocab 50304), M=16 micro-batches per iteration, split
(1,1,1): params, checkpoints and the fp32 optimizer state (master, m, v) live
in pinned host DRAM, and the plan's CpuStep runs where the state lives — on
the host cores (opt_tier 3, the reference's resource model,
proj/src/simulator.cpp:24-43): the GradAccum D2H lands the fp32 gradient in
DRAM, the AVX2 Adam writes the bf16 params straight into their host copy;
alpha=0.2, bf16.  The iteration roofline adds the host-DRAM term (30 B per
stepped element over the measured host copy bandwidth).  Variants:
`gpt1.3b-stream-opt` (state streamed through HBM and stepped by the fused
GPU kernel, 26 B/element of extra PCIe, counted in e2e and the roofline) and
`gpt1.3b-hbm-opt` (state resident in HBM).  GPT-65B,
the metric's headline model, does not fit this box (196 GB DRAM / 80 GB
disk); `--config gpt65b-8layer` runs its layer geometry on an 8-layer slice
with the optimizer state split between pinned DRAM and the NVMe file.

--impl reference times the reference CPU path on the host cores: the
reference's offsim carries no training arithmetic, so the timed CPU
implementation is the C oracle port (oracle/gs_oracle.c, fp32, OpenMP) —
each step one layer's forward + recompute + backward at b=1, s=2048, plus the
tied LM head timed once — extrapolated to one training step of the workload.

Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun
re-launches itself under torch.distributed.run).  ZeRO-3 data parallelism
inside the executor: each rank runs its own M micro-batches (global batch
grows with N: scaling "weak"), owns 1/N of every layer's params / grads /
optimizer state, all-gathers layer shards before each stage and
reduce-scatters the fp32 layer gradient after it; rank 0 reports
max-over-ranks time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

# one metric string for both arms (the driver computes the ours/reference ratio)
METRIC = "tokens/sec (GPT-1.3B training, vertical schedule + alpha-delayed optimizer step, BASELINE configs[1])"

OPT_TIERS = {0: "auto", 1: "HBM", 2: "pinned host DRAM, streamed through HBM per step",
             3: "pinned host DRAM, stepped by the host cores (the reference's CpuStep)"}

CONFIGS = {
    # name: (N, h, heads, s, b, vocab, M, split, alpha, opt_tier, ssd_ring_layers)
    # BASELINE configs[1] as written: everything CPU-resident in pinned DRAM
    "gpt1.3b": (24, 2048, 16, 2048, 2, 50304, 16, (1.0, 1.0, 1.0), 0.2, 3, 8),
    # the same with the CPU-resident optimizer fraction held in HBM instead
    "gpt1.3b-hbm-opt": (24, 2048, 16, 2048, 2, 50304, 16, (1.0, 1.0, 1.0), 0.2, 1, 8),
    "gpt1.3b-stream-opt": (24, 2048, 16, 2048, 2, 50304, 16, (1.0, 1.0, 1.0), 0.2, 2, 8),
    "gpt1.3b-host-opt": (24, 2048, 16, 2048, 2, 50304, 16, (1.0, 1.0, 1.0), 0.2, 3, 8),
    "gpt1.3b-ssd-opt": (24, 2048, 16, 2048, 2, 50304, 16, (1.0, 1.0, 0.0), 0.2, 3, 8),
    # BASELINE configs[2] shape on this box (196 GB DRAM, 80 GB disk): half of
    # the optimizer state (75.5 GB) on the NVMe tier, the other half in DRAM
    "gpt13b-nvme": (40, 5120, 40, 2048, 2, 50304, 16, (1.0, 1.0, 0.5), 0.2, 3, 4),
    # GPT-65B layer geometry (h = 8192, 64 heads, b = 2, M = 32: BASELINE
    # configs[3] per rank, split (1,1,0.5)) on an 8-layer slice: the optimizer
    # state half in pinned DRAM, half on the NVMe file (38.7 GB), never in HBM,
    # stepped by the host cores; 4 layers of NVMe staging.  The full 80-layer
    # model needs 773 GB of optimizer state (> this box)
    "gpt65b-8layer": (8, 8192, 64, 2048, 2, 50304, 32, (1.0, 1.0, 0.5), 0.2, 3, 4),
    # BASELINE configs[4] (GPT-175B, 1 GPU, split (1, 0, 0): params and the
    # whole optimizer state on the NVMe file, checkpoints in DRAM, b=1, M=32)
    # on a 2-layer slice of its layer geometry (h = 12288, 96 heads): 50.7 GB
    # on the NVMe file, the most this box's 80 GB disk holds with the probe's
    # scratch.  CpuStep on the host cores over the staged state
    "gpt175b-2layer": (2, 12288, 96, 2048, 1, 50304, 32, (1.0, 0.0, 0.0), 0.2, 3, 2),
    "tiny": (4, 64, 4, 32, 2, 128, 4, (1.0, 1.0, 0.5), 0.25, 2, 8),
}


def make_tokens(V, iters, M, b, s, seed):
    """Synthetic token ids, uniform in [0, V), [iters][M][b][s+1]."""
    return np.random.default_rng(seed).integers(0, V, size=(iters, M, b, s + 1), dtype=np.int32)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        loaded = [x for x in sm if x > 500] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for name, v in zip(names, r[3:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)  # gloo: the timing plumbing, not the data path
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def pcie_bandwidth(torch, nbytes=1 << 30):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            fn()
        b.record()
        torch.cuda.synchronize()
        out[name] = 3 * nbytes / (a.elapsed_time(b) / 1e3)
    del h, d
    return out


def cpu_model() -> str:
    """The host CPU's model name (/proc/cpuinfo) and nproc, reported next to CPU numbers."""
    name = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                name = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{name}, nproc {os.cpu_count()}"


_HEAD_S = {}


def cpu_sample(cfg_name: str, head: bool = False):
    """Time the oracle port (fp32 C, OpenMP, all host threads) on one layer's
    forward + recompute-and-backward at b=1 and the workload's full sequence
    (or, head=True, the tied LM head: final LN, logits, CE, both grads).
    Returns (seconds, threads)."""
    import oracle_bindings as ob
    N, h, H, s, b, V = CONFIGS[cfg_name][:6]
    g = ob.Geometry(n_layers=N, hidden=h, heads=H, seq=s, mb_size=1, vocab=V)
    cfg = g.cfg()
    lib = ob.oracle()
    rng = np.random.default_rng(0)
    f = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
    x = rng.standard_normal(s * h).astype(np.float32)
    dx = np.empty_like(x)
    if head:
        wte = (rng.standard_normal(V * h) * 0.02).astype(np.float32)
        dwte = np.zeros_like(wte)
        tok = rng.integers(0, V, s + 1, dtype=np.int32)
        t0 = time.perf_counter()
        lib.gso_head(C.byref(cfg), f(wte), f(x), tok.ctypes.data_as(C.POINTER(C.c_int32)), C.c_float(1.0 / s),
                     f(dx), f(dwte))
        return time.perf_counter() - t0, lib.gso_num_threads()
    w = (rng.standard_normal(12 * h * h) * 0.02).astype(np.float32)
    dy = rng.standard_normal(s * h).astype(np.float32) * 0.01
    y = np.empty_like(x)
    dw = np.zeros_like(w)
    t0 = time.perf_counter()
    lib.gso_layer_fwd(C.byref(cfg), f(w), f(x), f(y))
    lib.gso_layer_bwd(C.byref(cfg), f(w), f(x), f(dy), f(dx), f(dw))
    return time.perf_counter() - t0, lib.gso_num_threads()


def cpu_step_estimate(cfg_name: str, t_layer: float):
    """Extrapolate one training step of the workload from a layer sample and
    the (cached) head sample: M*b sequences x (N layers + head)."""
    N, h, H, s, b, V, M = CONFIGS[cfg_name][:7]
    if cfg_name not in _HEAD_S:
        _HEAD_S[cfg_name] = cpu_sample(cfg_name, head=True)[0]
    t_step = M * b * (N * t_layer + _HEAD_S[cfg_name])
    desc = (f"oracle C fp32 port: per step 1 layer fwd + recompute + bwd at b=1, s={s}, h={h} timed, the tied LM "
            f"head (V={V}) timed once ({_HEAD_S[cfg_name]:.2f} s); step = M*b*(N*t_layer + t_head) with M={M}, b={b}, "
            f"N={N}; embedding and the Adam step (< 0.1%) excluded")
    return t_step, M * b * s, desc


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    for _ in range(args.warmup if args.config == "tiny" else 0):
        cpu_sample(args.config)
    steps, threads = [], 1
    for _ in range(args.steps):
        dt, threads = cpu_sample(args.config)
        steps.append(cpu_step_estimate(args.config, dt))
    t_step = float(np.mean([t for t, _, _ in steps]))
    toks, desc = steps[0][1], steps[0][2]
    value = toks / t_step
    line = {"impl": "reference", "metric": metric(args),
            "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3,
            "ms_per_step_note": "extrapolated CPU time of one training step of the workload (not the sample's)",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(args),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": desc,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def metric(args):
    if args.schedule == "horizontal":
        return f"tokens/sec ({args.config} training, horizontal schedule (the ablation baseline))"
    if args.config == "gpt1.3b":
        return METRIC
    return f"tokens/sec ({args.config} training, vertical schedule + alpha-delayed optimizer step)"


def config_dict(args):
    N, h, H, s, b, V, M, split, alpha, tier, ring = CONFIGS[args.config]
    M = args.microbatches or M
    ring = args.ssd_ring or ring
    tier = tier if args.opt_tier < 0 else args.opt_tier
    alpha = args.alpha if args.alpha >= 0 else alpha
    alpha = alpha if args.schedule == "vertical" else 0.0
    place = (f"CPU-resident fractions (split) in pinned host DRAM, the rest on the NVMe file; "
             f"CPU-resident optimizer state: {OPT_TIERS[tier]}")
    return {"workload": f"{args.config}: GPT N={N} h={h} heads={H} s={s} b={b} vocab={V}, {args.schedule} schedule, "
                        f"M={M} micro-batches/iteration, split(x_ckpt,x_param,x_opt)={split}, alpha={alpha}; {place}",
            "schedule": args.schedule, "opt_tier": OPT_TIERS[tier],
            "global_batch": M * b * max(args.gpus, 1), "seq_len": s, "microbatches": M, "alpha": alpha,
            "split": list(split), "ssd_ring_layers": ring, "parallelism": f"zero3-dp{args.gpus}" if args.gpus > 1 else "single",
            "l2": "working set (params / optimizer state streamed, GBs per iteration) >> 126 MB L2; no flush needed"}


def calibrate_and_simulate(gs, eng, plan, model, tokens, K, dev_ms):
    """§8(f): feed the executor's measured per-task times into the
    reference's MachineSpec and compare simulate()'s predicted iteration time
    (proj/src/simulator.cpp:77) with the measured one."""
    import numpy as np
    eng.set_trace(True)
    rep = eng.run(tokens, iterations=2)
    eng.set_trace(False)
    tasks = [plan.task(i) for i in range(len(plan))]
    last = [r for r in rep.trace if r["iteration"] == 1]
    def mean_ms(kind):
        d = [r["t_end_ms"] - r["t_start_ms"] for r in last if tasks[r["task"]]["kind"] == kind]
        return float(np.mean(d)) if d else 0.0
    steps = [(r, tasks[r["task"]]) for r in last if tasks[r["task"]]["kind"] == "cpu_step"]
    el = sum(t["elements"] for _, t in steps)
    step_ms = sum(r["t_end_ms"] - r["t_start_ms"] for r, _ in steps)
    xfer = {}
    for r in last:
        t = tasks[r["task"]]
        if t["kind"] == "xfer":
            a = xfer.setdefault(t["link"], [0, 0.0])
            a[0] += t["bytes"]
            a[1] += r["t_end_ms"] - r["t_start_ms"]
    bw = {k: (v[0] / (v[1] / 1e3) if v[1] > 0 else 1e12) for k, v in xfer.items()}
    machine = gs.MachineSpec(gpu_mem_bytes=180 << 30, cpu_usable_dram_bytes=190 << 30,
                             pcie_h2d_bw=bw.get("H2D", 55e9), pcie_d2h_bw=bw.get("D2H", 55e9),
                             ssd_read_bw=bw.get("SSD_read", 1e12), ssd_write_bw=bw.get("SSD_write", 1e12),
                             fwd_compute_time_per_layer_per_mb=mean_ms("fwd") / 1e3,
                             bwd_compute_time_per_layer_per_mb=mean_ms("bwd") / 1e3,
                             cpu_step_throughput=el / (step_ms / 1e3) if step_ms > 0 else 1e12,
                             fixed_overhead_time=mean_ms("fixed_ops") / 1e3, num_gpus=1,
                             gpu_working_set_bytes=1 << 30, ssd_duplex=True)
    sim = gs.simulate(plan, machine)
    measured = dev_ms / K
    # the planner (Algorithm 1, planner.cpp:72-201) on the same measured
    # constants: its projection of this configuration, and its own choice
    pd = plan.as_dict() if len(plan) < 20000 else None
    here = gs.solve_config(model, machine, pd["microbatches"], pd["alpha"]) if pd else None
    best = gs.find_optimal_config(model, machine)
    planner = {"this_config_projection_ms": here.iteration_estimate * 1e3 if here and here.feasible else None,
               "this_config_lp_split": [here.split.x_ckpt, here.split.x_param, here.split.x_opt] if here else None,
               "optimal": {"microbatches": best.num_microbatches, "alpha": best.alpha,
                           "split": [best.split.x_ckpt, best.split.x_param, best.split.x_opt],
                           "projected_iteration_ms": best.iteration_estimate * 1e3,
                           "projected_tokens_s": best.throughput_estimate * model.seq_len} if best.feasible else None}
    return {"method": "MachineSpec from this run's executor trace (mean task times, per-link achieved "
                      "bandwidth, Adam elements/s) -> offsim::simulate (proj/src/simulator.cpp:77)",
            "planner": planner,
            "predicted_iteration_ms": sim["iteration_time"] * 1e3, "measured_iteration_ms": measured,
            "gap": sim["iteration_time"] * 1e3 / measured - 1.0, "bound_class": sim["bound_class"],
            "utilization": sim["utilization"],
            "machine": {"fwd_ms": mean_ms("fwd"), "bwd_ms": mean_ms("bwd"), "fixed_ms": mean_ms("fixed_ops"),
                        "h2d_gbs": bw.get("H2D", 0) / 1e9, "d2h_gbs": bw.get("D2H", 0) / 1e9,
                        "adam_gelem_s": (el / (step_ms / 1e3) / 1e9) if step_ms > 0 else None}}


def run_ours(args):
    rank, world, local = dist_env()
    if world != args.gpus:  # before touching a device: a --gpus N line must come from N ranks
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world} ranks")
    import torch
    import torch.distributed as dist
    if world > 1:
        # one process per GPU; --share-gpu places every rank on the visible
        # device(s) round-robin (a functional check of the multi-rank path on
        # a smaller box: its numbers are not scaling results)
        ndev = torch.cuda.device_count()
        if local >= ndev and not args.share_gpu:
            raise SystemExit(f"bench: rank {rank} needs cuda:{local} but {ndev} GPU(s) are visible (--share-gpu)")
        torch.cuda.set_device(local % ndev)
        # gloo carries only the launcher plumbing (id broadcast, barriers,
        # max-over-ranks timing); the training collectives are the
        # executor's own peer-memory ones
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    import paper_2512_17570_b200 as gs
    N, h, H, s, b, V, M, split, alpha, tier, ring = CONFIGS[args.config]
    M = args.microbatches or M
    ring = args.ssd_ring or ring
    tier = tier if args.opt_tier < 0 else args.opt_tier
    alpha = args.alpha if args.alpha >= 0 else alpha
    model = gs.ModelSpec(N, h, H, s, b, 2, 4, 3, world)  # ZeRO-3 over the ranks
    if args.schedule == "horizontal":
        alpha = 0.0
        plan = gs.build_horizontal(model, M, gs.StorageSplit(*split))
    else:
        plan = gs.build_vertical(model, M, gs.StorageSplit(*split), alpha)
    nvme = os.environ.get("GS_NVME_DIR", "/tmp")
    comm_id = None
    if world > 1:  # rank 0 draws the peer-memory communicator id; the torch process group broadcasts it
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(gs.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        comm_id = bytes(idt.cpu().numpy().tobytes())
    eng = gs.Engine(plan, model, V, gs.AdamConfig(1e-4, 0.9, 0.95, 1e-8, 0.0), seed=1234,
                    device=torch.cuda.current_device(), nvme_dir=nvme, opt_tier=tier, profile=True, rank=rank,
                    world=world, comm_id=comm_id, ssd_ring_layers=ring, host_threads=args.host_threads)
    K, W = args.steps, args.warmup
    tokens = make_tokens(V, W + 2 * K, M, b, s, seed=7 + rank)
    # warm-up (untimed)
    eng.set_profiling(0)
    eng.run(tokens[:W])
    # timed region: one GEMM launch in 16 (per kernel class) is bracketed by
    # CUDA events on the compute stream for the live roofline
    eng.set_profiling(16)
    # device-resident tokens: `value`
    dtok = torch.tensor(tokens[W:W + K], device="cuda")
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        rep = eng.run(None, iterations=K, tokens_on_device=True, device_ptr=dtok.data_ptr())
    torch.cuda.synchronize()
    barrier(world)
    dev_ms = max_over_ranks(rep.total_ms, world)
    prof = eng.kernel_profile()
    eng.set_profiling(0)
    calib = None
    if args.calibrate and world == 1:
        calib = calibrate_and_simulate(gs, eng, plan, model, tokens[W:W + 2], K, dev_ms)
    # end-to-end through the public call: host tokens, losses read back
    barrier(world)
    t0 = time.perf_counter()
    rep_e2e = eng.run(tokens[W + K:W + 2 * K])
    e2e_wall = time.perf_counter() - t0
    e2e_ms = max_over_ranks(rep_e2e.total_ms, world)
    barrier(world)
    eng.close()
    if rank != 0:
        return
    tokens_per_step = M * b * s
    value = world * K * tokens_per_step / (dev_ms / 1e3)
    e2e_value = world * K * tokens_per_step / (e2e_ms / 1e3)
    hbm, tf_burst, tf_sust, src = peaks()
    # dominant kernel: the tcgen05 GEMM (fp32 accumulate, bf16 operands)
    gemm_flops, gemm_ms, gemm_sampled, gemm_all = prof.get("gemm", (0.0, 0.0, 0, 0))
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    # traffic: DRAM bytes per GEMM launch from the committed ncu launch list of
    # this command (profiles/, dram__bytes_read + write per launch), if present
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "round2", "gemm_traffic_r2q.json")
    if args.config == "gpt1.3b" and os.path.exists(tpath):
        t = json.load(open(tpath))
        traffic, traffic_src = t.get("gemm_dram_bytes_per_launch"), t.get("source")
    roof = {"bound": "tensor", "achieved": achieved, "peak": tf_sust, "unit": "TFLOP/s",
            "frac": achieved / tf_sust, "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read+write)",
            "traffic_source": traffic_src, "kernel": "tc_gemm_kernel (tcgen05, all layer GEMMs)",
            "launches_timed": gemm_sampled, "launches_total": gemm_all,
            "avg_launch_ms": gemm_ms / max(gemm_sampled, 1), "flops_per_launch": gemm_flops / max(gemm_sampled, 1),
            "method": "CUDA events around 1 in 16 of the forward / recompute tcgen05 GEMM launches (QKV, out-proj, "
                      "FC1+GELU, FC2+residual, LM head), which run alone on the compute stream; the backward GEMMs "
                      "overlap each other on two streams and are not timed; timed region",
            "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)"}
    span_flops, span_ms, span_n, _ = prof.get("gemm_span", (0.0, 0.0, 0, 0))
    if span_ms > 0:
        # the same launch population sampled without events (offset half a
        # stride): the kernel's own first-CTA-start .. last-CTA-exit span
        a_span = span_flops / (span_ms / 1e3) / 1e12
        roof.update({"achieved_kernel_span": a_span, "frac_kernel_span": a_span / tf_sust,
                     "avg_launch_ms_kernel_span": span_ms / span_n, "launches_kernel_span": span_n,
                     "kernel_span_method": "in-kernel %globaltimer (min over CTAs at work start after the PDL wait, "
                                           "max at CTA exit) on 1 in 16 of the same GEMM launches, none of them "
                                           "event-bracketed: an event pair between two PDL-chained kernels stops "
                                           "the next grid from launching under the previous one's drain, so the "
                                           "event-timed duration also carries that launch ramp"})
    # iteration roofline (north star): max of compute at peak and ledger bytes over measured links
    bw = pcie_bandwidth(torch)
    led, ext = rep.ledger, rep.extension
    flops_iter = N * 4 * (24 * h * h + 2 * s * h) * tokens_per_step
    t_comp = flops_iter / (tf_sust * 1e12)
    # PCIe: the plan's ledger plus the GPU optimizer's state streaming
    t_h2d = float(led[0].sum() + ext[0].sum()) / bw["h2d"]
    t_d2h = float(led[1].sum() + ext[1].sum()) / bw["d2h"]
    t_ssd, nvme = 0.0, None
    if float(led[2].sum() + led[3].sum()) > 0:
        # the NVMe tier's own bandwidth (O_DIRECT, 8 x 8 MiB in flight), both
        # directions concurrent as the SSD_R / SSD_W queues run
        out = (C.c_double * 3)()
        gs.check(gs.lib().gs_nvme_probe(os.environ.get("GS_NVME_DIR", "/tmp").encode(), C.c_uint64(4 << 30), out))
        nvme = {"write_gbs": out[0], "read_gbs": out[1], "concurrent_gbs_per_direction": out[2]}
        t_ssd = max(float(led[2].sum()), float(led[3].sum())) / (out[2] * 1e9)
    # host DRAM (OPT_HOST): the CpuStep bytes of the iteration — every layer's
    # P elements at 30 B (12 state in + 4 grad in + 12 state out + 2 bf16
    # param out) — over the measured multi-threaded host copy bandwidth
    t_host, host = 0.0, None
    if tier == 3:
        host = gs.host_probe()
        host["bytes_per_iteration"] = 30 * N * 12 * h * h // world
        t_host = host["bytes_per_iteration"] / (host["copy_gbs"] * 1e9)
    t_roof = max(t_comp, t_h2d, t_d2h, t_ssd, t_host)
    # the paper's narrower line-through-origin bound (roofline.cpp:8-22): only
    # the SSD-resident optimizer state's round trip, at the measured NVMe rate
    io_roof = None
    if nvme is not None:
        nv = nvme["concurrent_gbs_per_direction"] * 1e9
        mio = gs.MachineSpec(gpu_mem_bytes=180 << 30, cpu_usable_dram_bytes=190 << 30, pcie_h2d_bw=bw["h2d"],
                             pcie_d2h_bw=bw["d2h"], ssd_read_bw=nv, ssd_write_bw=nv,
                             fwd_compute_time_per_layer_per_mb=1e-3, bwd_compute_time_per_layer_per_mb=1e-3,
                             cpu_step_throughput=1e10, fixed_overhead_time=0.0, num_gpus=world,
                             gpu_working_set_bytes=1 << 30, ssd_duplex=True)
        io_roof = gs.io_roofline(model, mio, M * b, split[2]) * s
    ms_step = dev_ms / K
    line = {"metric": metric(args),
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens (uniform ids), random-init N(0,0.02) weights",
            "config": config_dict(args),
            "e2e": {"value": e2e_value, "unit": "tokens/s", "wall_s": e2e_wall,
                    "h2d_bytes_per_step": int(M * b * (s + 1) * 4 + led[0].sum() + rep.extension[0].sum()),
                    "d2h_bytes_per_step": int(8 + led[1].sum() + rep.extension[1].sum()),
                    "note": "host token ids copied to pinned memory and read by the GPU every step, losses read "
                            "back; PCIe bytes = the plan's offload ledger + the GPU optimizer's state / param "
                            "streaming (extension ledger), all inside the timed region"},
            "gpu_launches": rep.gpu_launches,
            "roofline": roof,
            "iteration_roofline": {"t_roof_ms": t_roof * 1e3, "t_measured_ms": ms_step, "frac": t_roof / (ms_step / 1e3),
                                   "t_compute_ms": t_comp * 1e3, "t_pcie_h2d_ms": t_h2d * 1e3,
                                   "t_pcie_d2h_ms": t_d2h * 1e3, "t_ssd_ms": t_ssd * 1e3, "nvme": nvme,
                                   "t_host_dram_ms": t_host * 1e3, "host_dram": host,
                                   "pcie_bytes": "ledger + extension (optimizer-state streaming) per direction",
                                   "pcie_h2d_gbs": bw["h2d"] / 1e9,
                                   "pcie_d2h_gbs": bw["d2h"] / 1e9, "flops_per_iteration": flops_iter,
                                   "compute_roofline_tokens_s": tokens_per_step / t_comp,
                                   "io_roofline_tokens_s": io_roof,
                                   "io_roofline_note": "offsim::io_roofline (roofline.cpp:8-22) x seq_len at the "
                                                       "measured NVMe rate; null when no optimizer state is on the "
                                                       "SSD (the bound is infinite)"},
            "offload_gb_per_iteration": {"ledger_h2d": float(led[0].sum()) / 1e9, "ledger_d2h": float(led[1].sum()) / 1e9,
                                         "ssd_read": float(led[2].sum()) / 1e9, "ssd_write": float(led[3].sum()) / 1e9,
                                         "extension_h2d": float(rep.extension[0].sum()) / 1e9,
                                         "extension_d2h": float(rep.extension[1].sum()) / 1e9},
            "ledger_equals_plan": bool(np.array_equal(led, gs.plan_traffic(plan))),
            "kernel_ms_per_step": {k: v[1] * v[3] / max(v[2], 1) / K for k, v in prof.items() if k != "gemm_span"},
            "kernel_ms_note": "1 launch in 16 per class bracketed by CUDA events, extrapolated; event overhead "
                              "inflates short kernels (LayerNorm ~10 us); device-time shares: profiles/ launch list",
            "losses": rep.losses,
            "model_vs_measured": calib,
            "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        dt, threads = cpu_sample(args.config)
        t_step, toks, desc = cpu_step_estimate(args.config, dt)
        line["cpu_baseline"] = {"value": toks / t_step, "unit": "tokens/s", "cores": threads, "kind": "port",
                                "sample": desc, "cpu": cpu_model()}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpt1.3b", choices=sorted(CONFIGS))
    ap.add_argument("--microbatches", type=int, default=0)
    ap.add_argument("--alpha", type=float, default=-1.0, help="override the config's delay ratio")
    ap.add_argument("--schedule", default="vertical", choices=["vertical", "horizontal"],
                    help="horizontal = the micro-batch-major ablation baseline (BASELINE configs[1])")
    ap.add_argument("--opt-tier", type=int, default=-1, choices=[-1, 0, 1, 2, 3],
                    help="override the config's optimizer tier (" + ", ".join(f"{k} {v}" for k, v in OPT_TIERS.items()) + ")")
    ap.add_argument("--ssd-ring", type=int, default=0, help="override the config's ssd_ring_layers (pinned staging slots)")
    ap.add_argument("--host-threads", type=int, default=0,
                    help="host-core optimizer threads per rank (0: hardware threads - 4, split over the node's ranks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--calibrate", type=int, default=1, help="calibrate offsim::simulate from the trace")
    ap.add_argument("--share-gpu", action="store_true",
                    help="N > 1 on fewer GPUs: ranks share devices (functional check, not a scaling number)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
