"""Sustained (power-capped) GEMM throughput: one GPT-1.3B layer's forward GEMM
sequence (QKV, out-proj + residual, FC1 + GELU, FC2 + residual) back to back
for ~3 s, ours vs cuBLAS (torch.matmul) on the same shapes, with the SM clock
sampled by nvidia-smi during each run.  Answers whether the in-step GEMM rate
(bench.py roofline.achieved) is the kernels' sustained rate or lost in-step."""
import ctypes as C
import json
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402

lib = gs.lib()
d = torch.device("cuda:0")
T, h = 4096, 2048
p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
shapes = [(T, 3 * h, h, 0), (T, h, h, 1), (T, 4 * h, h, 3), (T, h, 4 * h, 1)]
bufs = []
for M, N, K, epi in shapes:
    A = torch.randn(M * K, device=d).bfloat16()
    B = torch.randn(N * K, device=d).bfloat16()
    Cc = torch.empty(M * N, device=d, dtype=torch.bfloat16)
    R = torch.randn(M * N, device=d).bfloat16() if epi == 1 else None
    G = torch.empty(M * N, device=d, dtype=torch.bfloat16) if epi == 3 else None
    bufs.append((M, N, K, epi, A, B, Cc, R, G, A.view(M, K), B.view(N, K).t()))
flops = sum(2 * M * N * K for M, N, K, *_ in bufs)


def ours():
    for M, N, K, epi, A, B, Cc, R, G, *_ in bufs:
        gs.check(lib.gs_gemm(1, M, N, K, p(A), 1, p(B), 1, p(Cc), p(R), p(G), epi, None))


def ours_plain():  # no fused epilogue (bf16 C only), as cuBLAS
    for M, N, K, epi, A, B, Cc, R, G, *_ in bufs:
        gs.check(lib.gs_gemm(1, M, N, K, p(A), 1, p(B), 1, p(Cc), None, None, 0, None))


def cublas():
    for *_, A2, B2 in bufs:
        A2 @ B2


def clocks():
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip().split(",")
    return float(out[0]), float(out[1])


for name, fn in (("ours", ours), ("cublas", cublas), ("ours_plain", ours_plain), ("ours", ours), ("cublas", cublas),
                 ("ours_plain", ours_plain)):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    reps = 8000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    samples = []
    while not e1.query():
        samples.append(clocks())
        time.sleep(0.1)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    sm = sorted(s[0] for s in samples)
    pw = sorted(s[1] for s in samples)
    print(json.dumps({"impl": name, "seconds": ms / 1e3, "tflops": flops * reps / ms / 1e9,
                      "sm_mhz_median": sm[len(sm) // 2] if sm else None, "power_w_median": pw[len(pw) // 2] if pw else None}),
          flush=True)
