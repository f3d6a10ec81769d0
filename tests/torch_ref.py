"""TEST INFRASTRUCTURE ONLY — a plain PyTorch restatement of the training
math the executor runs, for parity checks at production geometries.

The C oracle (oracle/gs_oracle.c) is the pinned CPU checker, but at the
BASELINE layer geometries (h = 2048 / 5120 / 8192, s = 2048) one iteration of
it takes minutes on the host.  This module states the same model in torch
(the restatement tools/make_golden.py pins the oracle with):
pre-LN GPT block with exactly 12h^2 parameters [Wqkv | Wo | W1 | W2] (each
[out][in], model.cpp:29), non-affine LayerNorm (eps 1e-5), causal softmax
attention, tanh-GELU, tied embedding / LM head with learned positions, mean
cross-entropy over b*s tokens and M micro-batches, Adam with bias correction
(step t = iteration + 1).  The vertical schedule's alpha-delayed step applies
the same update, so a plain loop is the reference for
every plan.  Run in fp32 on the GPU (TF32 off) it checks the bf16 tcgen05
path and the fp32 parity mode at the real shapes; tests/test_torch_ref.py
pins it against tests/golden/tiny_golden.npz (torch fp64) and the C oracle.

Only tests/ import this module.
"""
from __future__ import annotations

import math

import numpy as np


# --------------------------------------------------------------- data / init
def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def stream_key(seed, stream):
    with np.errstate(over="ignore"):
        return splitmix64(np.uint64(seed) ^ splitmix64(np.uint64(stream) + np.uint64(0x632BE59BD9B4E019)))


def normal_at(seed, stream, idx):
    """N(0,1) sample `idx` of stream `stream` (oracle gso_normal)."""
    key = stream_key(seed, stream)
    i = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        a = splitmix64(key + np.uint64(2) * i)
        b = splitmix64(key + np.uint64(2) * i + np.uint64(1))
    u1 = ((a >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def layer_init_at(N, h, seed, layer, idx):
    """Initial master weight of elements `idx` of layer `layer` (gso_init_layer)."""
    idx = np.asarray(idx, dtype=np.int64)
    h2 = h * h
    out_proj = ((idx >= 3 * h2) & (idx < 4 * h2)) | (idx >= 8 * h2)
    std = np.where(out_proj, 0.02 / math.sqrt(2.0 * N), 0.02)
    return (std * normal_at(seed, 100 + layer, idx)).astype(np.float32)


def tokens(V, b, s, M, iteration, seed=1234):
    """Token ids of one iteration, [M][b][s+1] (gso_make_tokens)."""
    key = stream_key(seed, 1000000 + iteration)
    i = np.arange(M * b * (s + 1), dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = splitmix64(key + i)
    return (x % np.uint64(V)).astype(np.int32).reshape(M, b, s + 1)


# ---------------------------------------------------------------------- model
def _ln(torch, x):
    return torch.nn.functional.layer_norm(x, x.shape[-1:], eps=1e-5)


def layer_fwd(torch, x, w, h, H):
    b, s, _ = x.shape
    d = h // H
    h2 = h * h
    wqkv = w[:3 * h2].view(3 * h, h)
    wo = w[3 * h2:4 * h2].view(h, h)
    w1 = w[4 * h2:8 * h2].view(4 * h, h)
    w2 = w[8 * h2:].view(h, 4 * h)
    qkv = _ln(torch, x) @ wqkv.T
    q, k, v = (t.reshape(b, s, H, d).transpose(1, 2) for t in qkv.split(h, dim=-1))
    mask = torch.ones(s, s, dtype=torch.bool, device=x.device).triu(1)
    outs = []
    # one head group at a time bounds the [s][s] score memory at h = 8192
    step = max(1, min(H, 16))
    for j in range(0, H, step):
        att = (q[:, j:j + step] @ k[:, j:j + step].transpose(-1, -2)) / math.sqrt(d)
        att = att.masked_fill(mask, float("-inf")).softmax(-1)
        outs.append(att @ v[:, j:j + step])
    o = torch.cat(outs, dim=1).transpose(1, 2).reshape(b, s, h)
    x1 = x + o @ wo.T
    g = torch.nn.functional.gelu(_ln(torch, x1) @ w1.T, approximate="tanh")
    return x1 + g @ w2.T


def train(geom, adam, layers0, fixed0, toks, device="cpu", dtype="float32", checkpoint=True, autocast_bf16=False):
    """Plain-loop training of `toks` [iters][M][b][s+1] from the given fp32
    master weights.  Returns dict(losses, layers, fixed, m, v, fm, fv) as
    numpy float32 (losses float64).  autocast_bf16: the forward / backward
    under torch.autocast(bfloat16) (bf16 GEMMs with fp32 accumulation, fp32
    masters, gradients and Adam) — torch's own mixed-precision deviation from
    fp32, the yardstick for the executor's bf16 path."""
    import contextlib

    import torch
    import torch.utils.checkpoint as ckpt
    amp = (lambda: torch.autocast(device_type=device if device != "cpu" else "cpu", dtype=torch.bfloat16)) \
        if autocast_bf16 else contextlib.nullcontext

    N, h, H, s, V = geom.n_layers, geom.hidden, geom.heads, geom.seq, geom.vocab
    dt = getattr(torch, dtype)
    W = [torch.tensor(np.asarray(layers0[l]), dtype=dt, device=device).requires_grad_(True) for l in range(N)]
    F = torch.tensor(np.asarray(fixed0), dtype=dt, device=device).requires_grad_(True)
    params = W + [F]
    state = [(torch.zeros_like(p), torch.zeros_like(p)) for p in params]
    iters, M = toks.shape[0], toks.shape[1]
    losses = []
    for it in range(iters):
        for p in params:
            p.grad = None
        total = 0.0
        for m in range(M):
            t = torch.tensor(toks[it, m], dtype=torch.long, device=device)
            wte = F[:V * h].view(V, h)
            wpe = F[V * h:].view(s, h)
            with amp():
                x = wte[t[:, :s]] + wpe[None, :, :]
                for l in range(N):
                    # recompute-from-checkpoint, as the executor does (also bounds memory)
                    x = ckpt.checkpoint(layer_fwd, torch, x, W[l], h, H, use_reentrant=False) if checkpoint else \
                        layer_fwd(torch, x, W[l], h, H)
                logits = _ln(torch, x) @ wte.T
            logits = logits.float() if autocast_bf16 else logits
            loss = torch.nn.functional.cross_entropy(logits.reshape(-1, V), t[:, 1:].reshape(-1))
            (loss / M).backward()
            total += float(loss.item())
            del logits, loss, x
        losses.append(total / M)
        with torch.no_grad():
            b1, b2, lr, eps, wd = adam["beta1"], adam["beta2"], adam["lr"], adam["eps"], adam["weight_decay"]
            bc1, bc2 = 1 - b1 ** (it + 1), 1 - b2 ** (it + 1)
            for p, (m_, v_) in zip(params, state):
                g = p.grad
                m_.mul_(b1).add_((1 - b1) * g)
                v_.mul_(b2).add_((1 - b2) * g * g)
                p.sub_(lr * ((m_ / bc1) / ((v_ / bc2).sqrt() + eps) + wd * p))
    f32 = lambda x: x.detach().float().cpu().numpy()  # noqa: E731
    return dict(losses=np.array(losses, np.float64), layers=np.stack([f32(w) for w in W]), fixed=f32(F),
                m=np.stack([f32(a) for a, _ in state[:N]]), v=np.stack([f32(b) for _, b in state[:N]]),
                fm=f32(state[N][0]), fv=f32(state[N][1]))
