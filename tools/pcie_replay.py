"""Replay one forward stage's PCIe pattern without the layer kernels: the
compute stream runs 16 "tasks" (spin kernels of the measured 0.45 ms, or the
real tcgen05 FC1 GEMM x4 when argv[1] == "gemm"); D2H offloads each task's
16.8 MB checkpoint after it; H2D reloads 15 checkpoints back to back, then
the next layer's 100 MB of parameters in 16 pieces.  Per-copy rates with
CUDA events, as the executor trace records them."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
MB = 1 << 20
ck = 2 * 2048 * 2048 * 2
pp = 6291456
h_ck = torch.empty(32 * ck, dtype=torch.uint8, pin_memory=True)
h_pp = torch.empty(16 * pp, dtype=torch.uint8, pin_memory=True)
d_ck = torch.empty(32 * ck, dtype=torch.uint8, device="cuda")
d_pp = torch.empty(16 * pp, dtype=torch.uint8, device="cuda")
sc, sh, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
mode = sys.argv[1] if len(sys.argv) > 1 else "spin"
if mode == "gemm":
    import paper_2512_17570_b200 as gs
    lib = gs.lib()
    M, N, K = 4096, 8192, 2048
    A = torch.randn(M * K, device="cuda").bfloat16(); B = torch.randn(N * K, device="cuda").bfloat16()
    Cc = torch.empty(M * N, device="cuda", dtype=torch.bfloat16); G = torch.empty_like(Cc)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def task():
    if mode == "gemm":
        for _ in range(4):
            gs.check(lib.gs_gemm(1, M, N, K, p(A), 1, p(B), 1, p(Cc), None, p(G), 3, C.c_void_p(sc.cuda_stream)))
    else:
        torch.cuda._sleep(int(0.45e-3 * 1.6e9))


def ev():
    return torch.cuda.Event(enable_timing=True)


def stage():
    rec = []
    t0 = ev(); t0.record(sc); sh.wait_event(t0); sd.wait_event(t0)
    with torch.cuda.stream(sh):
        for k in range(15):
            a, b = ev(), ev(); a.record(sh)
            d_ck[k * ck:(k + 1) * ck].copy_(h_ck[k * ck:(k + 1) * ck], non_blocking=True)
            b.record(sh); rec.append(("h2d_ckpt", a, b, ck))
        for k in range(16):
            a, b = ev(), ev(); a.record(sh)
            d_pp[k * pp:(k + 1) * pp].copy_(h_pp[k * pp:(k + 1) * pp], non_blocking=True)
            b.record(sh); rec.append(("h2d_param", a, b, pp))
    for k in range(16):
        with torch.cuda.stream(sc):
            task()
            done = ev(); done.record(sc)
        sd.wait_event(done)
        with torch.cuda.stream(sd):
            a, b = ev(), ev(); a.record(sd)
            h_ck[(16 + k) * ck:(17 + k) * ck].copy_(d_ck[(16 + k) * ck:(17 + k) * ck], non_blocking=True)
            b.record(sd); rec.append(("d2h_ckpt", a, b, ck))
    torch.cuda.synchronize()
    out = {}
    for name, a, b, n in rec:
        out.setdefault(name, []).append(n / (a.elapsed_time(b) / 1e3) / 1e9)
    return {k: sorted(v)[len(v) // 2] for k, v in out.items()}


stage()
for _ in range(3):
    print(json.dumps({"mode": mode, "median_gbs": stage()}), flush=True)
