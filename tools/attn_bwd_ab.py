"""Attention backward timing at the GPT-1.3B shape (b=2, s=2048, H=16, d=128,
causal) — ours (prologue + tcgen05 kernel [+ dQ cast pass]) vs cuDNN SDPA
backward on the same box; CUDA events, best and median of 50 after warm-up.
Also checks dQ/dK/dV against torch fp32 autograd on the same inputs."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402

lib = gs.lib()
d = torch.device("cuda:0")
b, s, H, h = 2, 2048, 16, 2048


def p(t):
    return C.c_void_p(t.data_ptr())


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    ts.sort()
    return ts[0], ts[len(ts) // 2]


torch.manual_seed(0)
qkv = (torch.randn(b * s, 3 * h, device=d) * 0.5).bfloat16()
o = torch.empty(b * s, h, device=d).bfloat16()
lse = torch.empty(b * H * s, device=d)
gs.check(lib.gs_attention_fwd(1, p(qkv), p(o), p(lse), b, s, h, H, None))
dout = torch.randn(b * s, h, device=d).bfloat16()
dqkv = torch.zeros_like(qkv)
work = torch.empty(lib.gs_attention_bwd_workspace(b, s, h, H), dtype=torch.uint8, device=d)
run = lambda: gs.check(lib.gs_attention_bwd(1, p(qkv), p(o), p(lse), p(dout), p(dqkv), p(work), b, s, h, H, None))
best, med = timed(run)
fl = 2.5 * 4 * b * H * s * s / 2 * (h // H)
row = dict(kernel="attn_bwd", best_ms=best, median_ms=med,
           tflops_best=fl / best / 1e9)
# accuracy vs torch fp32 autograd
run()
torch.cuda.synchronize()
q, k, v = (qkv.float().view(b, s, 3, H, h // H)[:, :, i].transpose(1, 2).contiguous().requires_grad_(True)
           for i in range(3))
of = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
go = dout.float().view(b, s, H, h // H).transpose(1, 2)
gq, gk, gv = torch.autograd.grad(of, (q, k, v), go)
ref = torch.stack([g.transpose(1, 2).reshape(b * s, h) for g in (gq, gk, gv)], 1).reshape(b * s, 3 * h)
got = dqkv.float()
for i, name in enumerate(("dq", "dk", "dv")):
    sl = slice(i * h, (i + 1) * h)
    row[f"{name}_rel"] = float((got[:, sl] - ref[:, sl]).norm() / ref[:, sl].norm())
# repeatability: 20 more launches, dQ within reduce-order noise of the first
first = dqkv.clone()
worst = 0.0
for _ in range(20):
    run()
    torch.cuda.synchronize()
    worst = max(worst, float((dqkv.float() - first.float()).abs().max()))
row["repeat_max_abs_diff"] = worst
row["dkdv_repeat_bitexact"] = bool(torch.equal(dqkv[:, h:], first[:, h:]))
print(json.dumps(row), flush=True)
if os.environ.get("GS_AB_CUDNN", "1") == "1":
    from torch.nn.attention import SDPBackend, sdpa_kernel
    qq = torch.randn(b, H, s, h // H, device=d, dtype=torch.bfloat16, requires_grad=True)
    kk = torch.randn_like(qq, requires_grad=True)
    vv = torch.randn_like(qq, requires_grad=True)
    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
        out_t = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
        g = torch.randn_like(out_t)
        bf, mf = timed(lambda: torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True))
        bb, mb = timed(lambda: torch.autograd.grad(
            torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True), (qq, kk, vv), g))
    print(json.dumps(dict(kernel="cudnn_sdpa_bwd", best_ms=bb - bf, median_ms=mb - mf, note="fwd+bwd minus fwd")),
          flush=True)
