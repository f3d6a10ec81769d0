"""Throughput vs global batch and the schedule ablations on one B200
(BASELINE.json metric "tokens/sec vs global batch"; configs[1] and the
config-3 shape at GPT-1.3B scale).

Each row: a fresh executor, W untimed + K timed iterations with device-
resident tokens, tokens/s = K*M*b*s / (CUDA-event time), plus the plan's
offload bytes per iteration and the compute roofline fraction.
  vertical,  alpha=0.2, split (1,1,1), M in {1,2,4,8,16,32}   (batch sweep)
  vertical,  alpha=0,   M=16                                  (optimizer overlap off)
  horizontal,           M=16                                  (schedule ablation)
  vertical,  alpha=0.2/0, split (1,1,0), M=16                 (optimizer state on NVMe)
Usage: python tools/sweep.py [--quick] > gpurun_out/sweep.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--tier", type=int, default=3, choices=[0, 1, 2, 3],
                    help="optimizer tier (bench.OPT_TIERS), every row")
    ap.add_argument("--model", default="gpt1.3b", choices=["gpt1.3b", "gpt13b"],
                    help="gpt13b: BASELINE configs[2] shape, half the Adam state on NVMe, M and alpha sweep")
    args = ap.parse_args()
    import torch
    import paper_2512_17570_b200 as gs
    from bench import OPT_TIERS, make_tokens
    torch.cuda.set_device(0)
    N, h, H, s, b, V = 24, 2048, 16, 2048, 2, 50304
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops_sustained", 1400.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1400.0
    rows = [("vertical", 0.2, (1, 1, 1), m) for m in ([1, 4, 16] if args.quick else [1, 2, 4, 8, 16, 32])]
    rows += [("vertical", 0.0, (1, 1, 1), 16), ("horizontal", 0.0, (1, 1, 1), 16)]
    rows += [("vertical", 0.2, (1, 1, 0), 16), ("vertical", 0.0, (1, 1, 0), 16)]
    if args.model == "gpt13b":
        # 75.5 GB of Adam state on the NVMe tier (this box: 80 GB disk, 196 GB DRAM)
        N, h, H = 40, 5120, 40
        rows = [("vertical", a, (1, 1, 0.5), m) for m in (8, 16, 32) for a in (0.2, 0.0)]
    model = gs.ModelSpec(N, h, H, s, b, 2, 4, 3, 1)
    for sched, alpha, split, M in rows:
        if sched == "horizontal":
            plan = gs.build_horizontal(model, M, gs.StorageSplit(*split))
        else:
            # the alpha-residency rule (schedule.cpp:293-305) caps alpha at small M:
            # take the largest feasible alpha <= the requested one
            for a in [alpha] + [x for x in (0.15, 0.1, 0.05, 0.02, 0.0) if x < alpha]:
                try:
                    plan = gs.build_vertical(model, M, gs.StorageSplit(*split), a)
                    alpha = a
                    break
                except gs.InfeasibleError:
                    continue
        tier = args.tier
        t0 = time.perf_counter()
        eng = gs.Engine(plan, model, V, gs.AdamConfig(1e-4, 0.9, 0.95, 1e-8, 0.0), seed=1234,
                        nvme_dir=os.environ.get("GS_NVME_DIR", "/tmp"), opt_tier=tier,
                        ssd_ring_layers=4 if args.model == "gpt13b" else 8)
        setup_s = time.perf_counter() - t0
        tokens = make_tokens(V, args.warmup + args.steps, M, b, s, seed=7)
        eng.run(tokens[:args.warmup])
        dtok = torch.tensor(tokens[args.warmup:], device="cuda")
        torch.cuda.synchronize()
        rep = eng.run(None, iterations=args.steps, tokens_on_device=True, device_ptr=dtok.data_ptr())
        eng.close()
        del dtok
        ms = rep.total_ms / args.steps
        tok = M * b * s
        flops = N * 4 * (24 * h * h + 2 * s * h) * tok
        led = rep.ledger
        print(json.dumps({
            "model": args.model, "schedule": sched, "alpha": alpha, "split": list(split), "microbatches": M,
            "global_batch": M * b, "opt_tier": OPT_TIERS[tier],
            "tokens_per_s": tok / (ms / 1e3), "ms_per_iteration": ms,
            "compute_roofline_frac": flops / (peak * 1e12) / (ms / 1e3),
            "offload_gb": {"h2d": float(led[0].sum()) / 1e9, "d2h": float(led[1].sum()) / 1e9,
                           "ssd_read": float(led[2].sum()) / 1e9, "ssd_write": float(led[3].sum()) / 1e9,
                           "ext_h2d": float(rep.extension[0].sum()) / 1e9,
                           "ext_d2h": float(rep.extension[1].sum()) / 1e9},
            "ssd_physical_gb": {"read": float(rep.physical[2].sum()) / 1e9,
                                "write": float(rep.physical[3].sum()) / 1e9},
            "ledger_equals_plan": bool(np.array_equal(led, gs.plan_traffic(plan))),
            "host_pinned_gb": rep.host_pinned_bytes / 1e9, "gpu_gb": rep.gpu_bytes / 1e9,
            "losses": rep.losses, "setup_s": setup_s}), flush=True)


if __name__ == "__main__":
    main()
