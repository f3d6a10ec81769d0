"""Launch one kernel of interest a few times at GPT-1.3B shapes, for ncu
--set full captures (tools/final_round.sh): qkv | fc1 | wgrad | attn_fwd |
attn_bwd | ln_fwd [h] | ln_bwd [h].  Three launches; profile with `-s 2 -c 1` to skip warm-up."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402

lib = gs.lib()
d = torch.device("cuda:0")
T, h, b, s, H = 4096, 2048, 2, 2048, 16
p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
what = sys.argv[1]
torch.manual_seed(0)
if what in ("qkv", "fc1", "wgrad"):
    M, N, K, ak, bk, epi = {"qkv": (T, 3 * h, h, 1, 1, 0), "fc1": (T, 4 * h, h, 1, 1, 3),
                            "wgrad": (4 * h, h, T, 0, 0, 2)}[what]
    A = torch.randn(M * K, device=d).bfloat16()
    B = torch.randn(N * K, device=d).bfloat16()
    Cc = torch.zeros(M * N, device=d, dtype=torch.float32 if epi == 2 else torch.bfloat16)
    G = torch.empty(M * N, device=d, dtype=torch.bfloat16) if epi == 3 else None
    for _ in range(3):
        gs.check(lib.gs_gemm(1, M, N, K, p(A), ak, p(B), bk, p(Cc), None, p(G), epi, None))
elif what.startswith("ln"):  # ln_fwd | ln_bwd [h]: LayerNorm at T rows (bwd with the residual accumulate)
    hh = int(sys.argv[2]) if len(sys.argv) > 2 else h
    x = torch.randn(T, hh, device=d).bfloat16()
    y = torch.empty_like(x)
    mean = torch.empty(T, device=d)
    rstd = torch.empty(T, device=d)
    for _ in range(3):
        gs.check(lib.gs_layernorm_fwd(1, p(x), p(y), p(mean), p(rstd), T, hh, None))
        if what == "ln_bwd":
            gs.check(lib.gs_layernorm_bwd(1, p(x), p(mean), p(rstd), p(y), p(y), T, hh, 1, None))
else:
    qkv = (torch.randn(b * s, 3 * h, device=d) * 0.5).bfloat16()
    o = torch.empty(b * s, h, device=d).bfloat16()
    lse = torch.empty(b * H * s, device=d)
    for _ in range(3 if what == "attn_fwd" else 1):
        gs.check(lib.gs_attention_fwd(1, p(qkv), p(o), p(lse), b, s, h, H, None))
    if what == "attn_bwd":
        dout = torch.randn(b * s, h, device=d).bfloat16()
        dqkv = torch.empty_like(qkv)
        work = torch.empty(lib.gs_attention_bwd_workspace(b, s, h, H), dtype=torch.uint8, device=d)
        for _ in range(3):
            gs.check(lib.gs_attention_bwd(1, p(qkv), p(o), p(lse), p(dout), p(dqkv), p(work), b, s, h, H, None))
torch.cuda.synchronize()
