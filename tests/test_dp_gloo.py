"""Data parallelism on CPU with gloo, world_size 2.

The executor's ZeRO-3 contract, restated with the numeric oracle's
arithmetic and torch.distributed collectives: each rank runs its own M
micro-batches (loss scale 1/(T*M*W)), the fp32 layer gradients are
reduce-scattered into ceil(P/W)-element shards, each rank steps only its
shard of the optimizer state, and the updated shards are all-gathered; the
tied embedding gradient is all-reduced.  Must equal single-process training
on all W*M micro-batches.  Shard layout = paper_2512_17570_b200.shard_range.
"""
import ctypes as C
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_bindings as ob

ADAM = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)
G = ob.Geometry(n_layers=2, hidden=64, heads=4, seq=32, mb_size=2, vocab=128)
M, W, ITERS = 2, 2, 2


def shard_range(P, world, rank):
    ps = -(-P // world)
    lo = min(P, rank * ps)
    return lo, min(P, lo + ps)


def f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def dp_worker(rank, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=W)
    lib = ob.oracle()
    cfg = G.cfg()
    adam = ob.GsoAdam(**ADAM)
    layers, fixed = ob.init_params(G)
    tokens = ob.make_tokens(G, ITERS, M * W)
    P, T, h = G.P, G.mb_size * G.seq, G.hidden
    lo, hi = shard_range(P, W, rank)
    m_s = np.zeros((G.n_layers, hi - lo), np.float32)
    v_s = np.zeros_like(m_s)
    fm, fv = np.zeros_like(fixed), np.zeros_like(fixed)
    scale = 1.0 / (T * M * W)
    for it in range(ITERS):
        grads = np.zeros_like(layers)
        fgrad = np.zeros_like(fixed)
        wte, wpe = fixed[:G.vocab * h], fixed[G.vocab * h:]
        for mb in range(M):
            tok = np.ascontiguousarray(tokens[it, rank * M + mb])
            xs = [np.empty(T * h, np.float32) for _ in range(G.n_layers + 1)]
            lib.gso_embed_fwd(C.byref(cfg), f32p(wte), f32p(wpe), i32p(tok), f32p(xs[0]))
            for l in range(G.n_layers):
                lib.gso_layer_fwd(C.byref(cfg), f32p(layers[l]), f32p(xs[l]), f32p(xs[l + 1]))
            d = np.empty(T * h, np.float32)
            dwte = fgrad[:G.vocab * h]
            lib.gso_head(C.byref(cfg), f32p(wte), f32p(xs[-1]), i32p(tok), C.c_float(scale), f32p(d), f32p(dwte))
            for l in reversed(range(G.n_layers)):
                lib.gso_layer_bwd(C.byref(cfg), f32p(layers[l]), f32p(xs[l]), f32p(d), f32p(d), f32p(grads[l]))
            fg = np.ascontiguousarray(fgrad)
            lib.gso_embed_bwd(C.byref(cfg), i32p(tok), f32p(d), f32p(fg), f32p(fg[G.vocab * h:]))
            fgrad = fg
        # reduce-scatter of each layer's fp32 gradient (all-reduce + own shard)
        gt = torch.from_numpy(grads)
        dist.all_reduce(gt)
        grads = gt.numpy()
        ft = torch.from_numpy(fgrad)
        dist.all_reduce(ft)
        fgrad = ft.numpy()
        ps = -(-P // W)
        for l in range(G.n_layers):
            p_shard = np.ascontiguousarray(layers[l, lo:hi])
            g_shard = np.ascontiguousarray(grads[l, lo:hi])
            ms, vs = np.ascontiguousarray(m_s[l]), np.ascontiguousarray(v_s[l])
            lib.gso_adam_step(C.byref(adam), f32p(p_shard), f32p(ms), f32p(vs), f32p(g_shard), C.c_longlong(hi - lo),
                              it + 1, C.c_float(1.0))
            m_s[l], v_s[l] = ms, vs
            # all-gather of the updated shards (padded to ceil(P/W))
            padded = torch.zeros(ps)
            padded[:hi - lo] = torch.from_numpy(p_shard)
            parts = [torch.zeros(ps) for _ in range(W)]
            dist.all_gather(parts, padded)
            layers[l] = torch.cat(parts)[:P].numpy()
        fx = np.ascontiguousarray(fixed)
        lib.gso_adam_step(C.byref(adam), f32p(fx), f32p(fm), f32p(fv), f32p(fgrad), C.c_longlong(fixed.size), it + 1,
                          C.c_float(1.0))
        fixed = fx
    if rank == 0:
        np.save(out + "_layers.npy", layers)
        np.save(out + "_fixed.npy", fixed)
    dist.destroy_process_group()


def test_shard_ranges_tile_each_layer():
    for P in (1, 7, 49152, 12 * 2048 * 2048 + 5):
        for world in (1, 2, 3, 8):
            spans = [shard_range(P, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_zero3_dp_gloo_world2_matches_single_process(tmp_path):
    out = str(tmp_path / "dp")
    port = 29500 + (os.getpid() % 1000)
    mp.spawn(dp_worker, args=(port, out), nprocs=W, join=True)
    layers0, fixed0 = ob.init_params(G)
    tokens = ob.make_tokens(G, ITERS, M * W)
    _, ref_layers, ref_fixed, _, _ = ob.train(G, ADAM, M * W, None, tokens, layers0, fixed0)
    got_l = np.load(out + "_layers.npy")
    got_f = np.load(out + "_fixed.npy")
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    assert rel(got_l, ref_layers) < 1e-5
    assert rel(got_f, ref_fixed) < 1e-5


def test_package_shard_range_agrees():
    pytest.importorskip("paper_2512_17570_b200")
    import paper_2512_17570_b200 as gs
    for P, world in ((49152, 2), (49153, 3), (12 * 2048 * 2048, 8)):
        for r in range(world):
            assert gs.shard_range(P, world, r) == shard_range(P, world, r)
