"""Quick throughput probe of the sm_100a kernels at GPT-1.3B shapes
(T = b*s = 4096, h = 2048) — CUDA events, warm-up, best of N."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402

lib = gs.lib()
d = torch.device("cuda:0")


def p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


T, h = 4096, 2048
rows = []
# attention fwd / bwd at b=2, s=2048, h=2048, H=16
b, s, H = 2, 2048, 16
qkv = torch.randn(b * s, 3 * h, device=d).bfloat16()
o = torch.empty(b * s, h, device=d).bfloat16()
lse = torch.empty(b * H * s, device=d)
ms = timed(lambda: gs.check(lib.gs_attention_fwd(1, p(qkv), p(o), p(lse), b, s, h, H, None)))
fl = 4 * b * H * s * s / 2 * (h // H)
rows.append(dict(kernel="attn_fwd", ms=ms, tflops=fl / ms / 1e9))
dout = torch.randn(b * s, h, device=d).bfloat16()
dqkv = torch.empty_like(qkv)
work = torch.empty(lib.gs_attention_bwd_workspace(b, s, h, H), dtype=torch.uint8, device=d)
ms = timed(lambda: gs.check(lib.gs_attention_bwd(1, p(qkv), p(o), p(lse), p(dout), p(dqkv), p(work), b, s, h, H, None)))
rows.append(dict(kernel="attn_bwd", ms=ms, tflops=2.5 * fl / ms / 1e9))
# LayerNorm fwd / bwd(+residual) at the 1.3B / 13B / 65B widths: the step's
# shape (T rows, L2-resident) and 16x rows at h = 2048 (HBM)
for h_ln, rows_ln in ((2048, T), (2048, 16 * T), (5120, T), (8192, T)):
    x = torch.randn(rows_ln, h_ln, device=d).bfloat16()
    y = torch.empty_like(x)
    mean = torch.empty(rows_ln, device=d)
    rstd = torch.empty(rows_ln, device=d)
    ms = timed(lambda: gs.check(lib.gs_layernorm_fwd(1, p(x), p(y), p(mean), p(rstd), rows_ln, h_ln, None)))
    rows.append(dict(kernel="ln_fwd", h=h_ln, rows=rows_ln, ms=ms, gbs=2 * x.numel() * 2 / ms / 1e6))
    ms = timed(lambda: gs.check(lib.gs_layernorm_bwd(1, p(x), p(mean), p(rstd), p(y), p(y), rows_ln, h_ln, 1, None)))
    rows.append(dict(kernel="ln_bwd_acc", h=h_ln, rows=rows_ln, ms=ms, gbs=4 * x.numel() * 2 / ms / 1e6))
    del x, y
# the same attention shapes through torch SDPA (cuDNN / flash backends) on
# this box, as the anchor for the tcgen05 kernels above
for backend in ("CUDNN_ATTENTION", "FLASH_ATTENTION"):
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel
        q = torch.randn(b, H, s, h // H, device=d, dtype=torch.bfloat16, requires_grad=True)
        k = torch.randn_like(q, requires_grad=True)
        v = torch.randn_like(q, requires_grad=True)
        with sdpa_kernel(getattr(SDPBackend, backend)):
            ms = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True))
            rows.append(dict(kernel=f"sdpa_{backend.lower()}_fwd", ms=ms, tflops=fl / ms / 1e9))
            out_t = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
            go = torch.randn_like(out_t)
            ms_fb = timed(lambda: torch.autograd.grad(
                torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True), (q, k, v), go))
            rows.append(dict(kernel=f"sdpa_{backend.lower()}_bwd", ms=ms_fb - ms, tflops=2.5 * fl / (ms_fb - ms) / 1e9,
                             note="fwd+bwd minus fwd"))
    except Exception as e:  # noqa: BLE001
        rows.append(dict(kernel=f"sdpa_{backend.lower()}", error=str(e)[:200]))
# one layer's FwdCompute / RecomputeAndBwd back to back (no executor): GPU ms
# per call and the host's enqueue ms per call
out = (C.c_double * 4)()
gs.check(lib.gs_layer_bench(1, 2, 2048, 2048, 16, 20, out))
rows.append(dict(kernel="layer_fwd", gpu_ms=out[0], host_enqueue_ms=out[1]))
rows.append(dict(kernel="layer_recompute_bwd", gpu_ms=out[2], host_enqueue_ms=out[3]))
if len(sys.argv) > 1 and sys.argv[1] == "attn":  # attention / LayerNorm / layer rows only
    for r in rows:
        print(json.dumps(r))
    sys.exit(0)
# GEMMs last: the GPT-65B shapes heat the GPU and would lower the clocks
# the attention / layer measurements see
for name, M, N, K, ak, bk, epi in [
        ("fwd_qkv", T, 3 * h, h, 1, 1, 0), ("fwd_fc1", T, 4 * h, h, 1, 1, 3), ("fwd_fc2", T, h, 4 * h, 1, 1, 1),
        ("dgrad_fc2", T, 4 * h, h, 1, 0, 0), ("wgrad_fc1", 4 * h, h, T, 0, 0, 2), ("sq8192", 8192, 8192, 8192, 1, 1, 0),
        # GPT-65B layer shapes (h = 8192): QKV, FC2 (K = 4h), FC1 weight gradient
        ("h8192_qkv", T, 3 * 8192, 8192, 1, 1, 0), ("h8192_fc2", T, 8192, 4 * 8192, 1, 1, 1),
        ("h8192_wgrad_fc1", 4 * 8192, 8192, T, 0, 0, 2)]:
    A = torch.randn(M * K, device=d).bfloat16()
    B = torch.randn(N * K, device=d).bfloat16()
    Cc = torch.empty(M * N, device=d, dtype=torch.float32 if epi == 2 else torch.bfloat16)
    R = torch.randn(M * N, device=d).bfloat16() if epi == 1 else None
    G = torch.empty(M * N, device=d, dtype=torch.bfloat16) if epi == 3 else None
    ms = timed(lambda: gs.check(lib.gs_gemm(1, M, N, K, p(A), ak, p(B), bk, p(Cc), p(R), p(G), epi, None)))
    rows.append(dict(gemm=name, M=M, N=N, K=K, ms=ms, tflops=2 * M * N * K / ms / 1e9))
# cuBLAS (torch.matmul) on the same GEMM shapes / operand majors, for context
for name, M, N, K, ak, bk in [("cublas_fwd_qkv", T, 3 * h, h, 1, 1), ("cublas_fwd_fc1", T, 4 * h, h, 1, 1),
                              ("cublas_fwd_fc2", T, h, 4 * h, 1, 1), ("cublas_dgrad_fc2", T, 4 * h, h, 1, 0),
                              ("cublas_wgrad_fc1", 4 * h, h, T, 0, 0), ("cublas_h8192_qkv", T, 3 * 8192, 8192, 1, 1),
                              ("cublas_h8192_fc2", T, 8192, 4 * 8192, 1, 1)]:
    A = torch.randn(M, K, device=d).bfloat16() if ak else torch.randn(K, M, device=d).bfloat16().t()
    B = torch.randn(N, K, device=d).bfloat16().t() if bk else torch.randn(K, N, device=d).bfloat16()
    ms = timed(lambda: A @ B)
    rows.append(dict(kernel=name, M=M, N=N, K=K, ms=ms, tflops=2 * M * N * K / ms / 1e9))
# torch reference matmul for context
A = torch.randn(8192, 8192, device=d).bfloat16()
B = torch.randn(8192, 8192, device=d).bfloat16()
ms = timed(lambda: A @ B)
rows.append(dict(kernel="torch_matmul_8192", ms=ms, tflops=2 * 8192 ** 3 / ms / 1e9))
for r in rows:
    print(json.dumps(r))
