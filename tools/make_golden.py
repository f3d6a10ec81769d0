"""Generate the golden vectors that pin the numeric oracle.

Independent arithmetic: torch float64 autograd on CPU (the reference carries
no training math).  The model, init and data stream are
restated here in numpy/torch (NOT loaded from the oracle): splitmix64 +
Box-Muller init, N(0,0.02) weights with the 1/sqrt(2N) output-projection
scale, uniform token ids.  Plain training loop: per iteration every
micro-batch forward+backward with fp64 gradient accumulation, then one Adam
step over all parameters — the semantics the vertical schedule with its
alpha-delayed step must reproduce.

Writes tests/golden/tiny_golden.npz.  Run:  python tools/make_golden.py
"""
from __future__ import annotations

import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "tiny_golden.npz")

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


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


def normal(seed, stream, n):
    key = stream_key(seed, stream)
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        a = splitmix64(key + np.uint64(2) * i)
        b = splitmix64(key + np.uint64(2) * i + np.uint64(1))
    u1 = ((a >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def init_layer(N, h, seed, layer):
    h2 = h * h
    z = normal(seed, 100 + layer, 12 * h2)
    std = np.full(12 * h2, 0.02)
    std[3 * h2:4 * h2] = 0.02 / np.sqrt(2.0 * N)
    std[8 * h2:] = 0.02 / np.sqrt(2.0 * N)
    return (std * z).astype(np.float32)


def init_fixed(V, s, h, seed):
    wte = (0.02 * normal(seed, 1, V * h)).astype(np.float32)
    wpe = (0.02 * normal(seed, 2, s * h)).astype(np.float32)
    return np.concatenate([wte, wpe])


def tokens(V, b, s, M, iteration, seed):
    key = stream_key(seed, 1000000 + iteration)
    i = np.arange(M * b * (s + 1), dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = splitmix64(key + i)
    return (x % np.uint64(V)).astype(np.int32).reshape(M, b, s + 1)


def ln(x):
    return torch.nn.functional.layer_norm(x, x.shape[-1:], eps=1e-5)


def layer_fwd(x, w, h, H):
    b, s, _ = x.shape
    d = h // H
    h2 = h * h
    wqkv = w[:3 * h2].view(3 * h, h)
    wo = w[3 * h2:4 * h2].view(h, h)
    w1 = w[4 * h2:8 * h2].view(4 * h, h)
    w2 = w[8 * h2:].view(h, 4 * h)
    qkv = ln(x) @ wqkv.T
    q, k, v = (t.view(b, s, H, d).transpose(1, 2) for t in qkv.split(h, dim=-1))
    att = (q @ k.transpose(-1, -2)) / np.sqrt(d)
    mask = torch.ones(s, s, dtype=torch.bool).triu(1)
    att = att.masked_fill(mask, float("-inf")).softmax(-1)
    o = (att @ v).transpose(1, 2).reshape(b, s, h)
    x1 = x + o @ wo.T
    g = torch.nn.functional.gelu(ln(x1) @ w1.T, approximate="tanh")
    return x1 + g @ w2.T


def train(cfg, adam, M, iters, seed=42, data_seed=1234):
    N, h, H, s, b, V = (cfg[k] for k in ("n_layers", "hidden", "heads", "seq", "mb_size", "vocab"))
    layers0 = np.stack([init_layer(N, h, seed, l) for l in range(N)])
    fixed0 = init_fixed(V, s, h, seed)
    W = [torch.tensor(layers0[l], dtype=torch.float64, requires_grad=True) for l in range(N)]
    F = torch.tensor(fixed0, dtype=torch.float64, requires_grad=True)
    params = W + [F]
    state = [(torch.zeros_like(p), torch.zeros_like(p)) for p in params]
    toks, losses = [], []
    for it in range(iters):
        tk = tokens(V, b, s, M, it, data_seed)
        toks.append(tk)
        for p in params:
            p.grad = None
        total = 0.0
        for m in range(M):
            t = torch.tensor(tk[m], dtype=torch.long)
            wte = F[:V * h].view(V, h)
            wpe = F[V * h:].view(s, h)
            x = wte[t[:, :s]] + wpe[None, :, :]
            for l in range(N):
                x = layer_fwd(x, W[l], h, H)
            logits = ln(x) @ wte.T
            loss = torch.nn.functional.cross_entropy(logits.reshape(-1, V), t[:, 1:].reshape(-1))
            (loss / M).backward()
            total += loss.item()
        losses.append(total / M)
        with torch.no_grad():
            b1, b2, lr, eps, wd = adam["beta1"], adam["beta2"], adam["lr"], adam["eps"], adam["weight_decay"]
            bc1, bc2 = 1 - b1 ** (it + 1), 1 - b2 ** (it + 1)
            for p, (m_, v_) in zip(params, state):
                g = p.grad
                m_.mul_(b1).add_((1 - b1) * g)
                v_.mul_(b2).add_((1 - b2) * g * g)
                p.sub_(lr * ((m_ / bc1) / ((v_ / bc2).sqrt() + eps) + wd * p))
    return (layers0, fixed0, np.stack(toks), np.array(losses),
            np.stack([w.detach().numpy() for w in W]), F.detach().numpy())


TINY = dict(n_layers=4, hidden=64, heads=4, seq=32, mb_size=2, vocab=128)
ADAM = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)
M, ITERS = 4, 3


def main():
    layers0, fixed0, toks, losses, layers, fixed = train(TINY, ADAM, M, ITERS)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(
        OUT, cfg=np.array([TINY[k] for k in ("n_layers", "hidden", "heads", "seq", "mb_size", "vocab")]),
        adam=np.array([ADAM[k] for k in ("lr", "beta1", "beta2", "eps", "weight_decay")]),
        microbatches=M, iters=ITERS, tokens=toks, init_layers=layers0, init_fixed=fixed0,
        losses=losses, final_layers=layers.astype(np.float32), final_fixed=fixed.astype(np.float32))
    print("wrote", OUT, "losses", losses)


if __name__ == "__main__":
    main()
