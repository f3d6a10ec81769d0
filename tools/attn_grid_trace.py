"""GS_ATTN_TRACE=1 run of the attention kernels at the GPT-1.3B shape
(b=2, s=2048, 16 heads, d=128): the grid schedule (span, CTAs per SM, mean
CTA time per blockIdx.y) and CTA (0,0)'s event timeline go to stderr."""
import ctypes as C
import os
import sys

import torch

os.environ["GS_ATTN_TRACE"] = "1"
sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402

lib = gs.lib()
d = torch.device("cuda:0")
b, s, h, H = 2, 2048, 2048, 16
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
qkv = torch.randn(b * s, 3 * h, device=d).bfloat16()
o = torch.empty(b * s, h, device=d).bfloat16()
lse = torch.empty(b * H * s, device=d)
dout = torch.randn(b * s, h, device=d).bfloat16()
dqkv = torch.empty_like(qkv)
work = torch.empty(lib.gs_attention_bwd_workspace(b, s, h, H), dtype=torch.uint8, device=d)
for it in range(3):
    print(f"=== fwd {it}", file=sys.stderr, flush=True)
    gs.check(lib.gs_attention_fwd(1, p(qkv), p(o), p(lse), b, s, h, H, None))
    torch.cuda.synchronize()
for it in range(3):
    print(f"=== bwd {it}", file=sys.stderr, flush=True)
    gs.check(lib.gs_attention_bwd(1, p(qkv), p(o), p(lse), p(dout), p(dqkv), p(work), b, s, h, H, None))
    torch.cuda.synchronize()
