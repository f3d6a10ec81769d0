"""The executor at the BASELINE layer geometries against a plain fp32 PyTorch
restatement of the same training (tests/torch_ref.py, pinned on CPU against
the torch-fp64 golden and the C oracle by tests/test_torch_ref.py).

Geometries (BASELINE.json configs):
  GPT-1.3B layer  h=2048, 16 heads, s=2048, b=2, vocab 50304, 2 layers
  GPT-13B layer   h=5120, 40 heads, s=2048, b=2, 1 layer
  GPT-65B layer   h=8192, 64 heads, s=2048, b=1, 1 layer
each as a vertical plan with the alpha-delayed step, M = 2 micro-batches
(alpha = 0.2 at GPT-1.3B; 0.1 / 0.04 at the one-layer 13B / 65B slices, the
largest delay ratios build_vertical's alpha-residency check admits there,
schedule.cpp:293-305), two iterations, the optimizer state in pinned host DRAM and
streamed through HBM (opt_tier 2, BASELINE configs[1]'s placement).

bf16 mode runs the production kernels (tcgen05 GEMMs, tcgen05 attention,
the LN / GELU / cross-entropy / fused Adam kernels).  Its distance from the
fp32 reference is judged against torch's own mixed precision on the same
inputs: tests/torch_ref.py under torch.autocast(bfloat16) (bf16 GEMMs, fp32
accumulation, fp32 masters / gradients / Adam).  Gates, per quantity
(measured values are printed; DESIGN.md §3 lists them):
  * per-step loss within 2e-3 relative of fp32;
  * Adam moments m, v after two steps (the layer weights and the embedding
    table; m is a linear combination of the two iterations' fp32-accumulated
    gradients): norm-relative distance from fp32 at most
    max(floor, 1.5 x torch-autocast's), floor 2e-2 for m and 4e-2 for v —
    the bf16 error grows with the contraction length (h = 8192: ~2.4e-2 for
    both implementations), so a fixed bound would either fail honest bf16
    or admit a broken gradient;
  * parameter update (w_final - w_init) within max(0.15, 1.5 x torch's) —
    Adam's first step is lr * sign(g) element-wise, so every gradient
    element whose bf16 and fp32 signs differ moves by 2 lr; a wrong
    gradient gives ~1.4.
fp32 mode (low_precision_bytes = 4) at the GPT-1.3B geometry holds the
north-star tolerances: loss 1e-3 relative, parameters after the steps (after
flush()) 1e-4 relative.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle_bindings as ob  # noqa: E402
import paper_2512_17570_b200 as gs  # noqa: E402
import torch_ref as tr  # noqa: E402

ADAM = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)

GEOMS = {
    "gpt1.3b": ob.Geometry(n_layers=2, hidden=2048, heads=16, seq=2048, mb_size=2, vocab=50304),
    "gpt13b": ob.Geometry(n_layers=1, hidden=5120, heads=40, seq=2048, mb_size=2, vocab=50304),
    "gpt65b": ob.Geometry(n_layers=1, hidden=8192, heads=64, seq=2048, mb_size=1, vocab=50304),
}


def need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run_both(g, lp, M=2, iters=2, alpha=0.2, split=(1, 1, 1), opt_tier=2):
    torch = need_gpu()
    model = gs.ModelSpec(g.n_layers, g.hidden, g.heads, g.seq, g.mb_size, lp, 4, 3, 1)
    plan = gs.build_vertical(model, M, gs.StorageSplit(*split), alpha)
    eng = gs.Engine(plan, model, g.vocab, gs.AdamConfig(**ADAM), seed=42, nvme_dir="/tmp", opt_tier=opt_tier)
    l0, f0 = eng.read_params()  # initial fp32 masters
    # the engine's init is the oracle's (bit-exact at the tiny geometry); spot-check it here
    rng = np.random.default_rng(0)
    for l in range(g.n_layers):
        idx = rng.integers(0, g.P, 4096)
        assert np.array_equal(l0[l, idx], tr.layer_init_at(g.n_layers, g.hidden, 42, l, idx))
    toks = np.stack([tr.tokens(g.vocab, g.mb_size, g.seq, M, it) for it in range(iters)])
    rep = eng.run(toks)
    eng.flush()
    l1, f1 = eng.read_params()
    m, v = eng.read_moments()
    fm, fv = eng.read_fixed_moments()
    eng.close()
    assert np.array_equal(rep.ledger, gs.plan_traffic(plan)), "executed ledger != plan ledger"
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    ref = tr.train(g, ADAM, l0, f0, toks, device="cuda", dtype="float32")
    torch.cuda.empty_cache()
    amp = None
    if lp == 2:
        amp = tr.train(g, ADAM, l0, f0, toks, device="cuda", dtype="float32", autocast_bf16=True)
        torch.cuda.empty_cache()
    out = dict(
        loss=float(np.max(np.abs(np.array(rep.losses) - ref["losses"]) / ref["losses"])),
        m=rel(m, ref["m"]), v=rel(v, ref["v"]), fm=rel(fm, ref["fm"]), fv=rel(fv, ref["fv"]),
        dw=rel(l1 - l0, ref["layers"] - l0), dfixed=rel(f1 - f0, ref["fixed"] - f0),
        w=rel(l1, ref["layers"]), fixed=rel(f1, ref["fixed"]))
    if amp is not None:
        out["torch_amp"] = dict(
            loss=float(np.max(np.abs(amp["losses"] - ref["losses"]) / ref["losses"])),
            m=rel(amp["m"], ref["m"]), v=rel(amp["v"], ref["v"]), fm=rel(amp["fm"], ref["fm"]),
            fv=rel(amp["fv"], ref["fv"]), dw=rel(amp["layers"] - l0, ref["layers"] - l0),
            dfixed=rel(amp["fixed"] - f0, ref["fixed"] - f0))
    print(f"\nparity h={g.hidden} lp={lp}: losses {rep.losses} ref {ref['losses'].tolist()} " +
          " ".join(f"{k}={x:.3e}" for k, x in out.items() if k != "torch_amp") +
          (" | torch autocast-bf16: " + " ".join(f"{k}={x:.3e}" for k, x in out["torch_amp"].items())
           if amp is not None else ""))
    return out


ALPHA = {"gpt1.3b": 0.2, "gpt13b": 0.1, "gpt65b": 0.04}


@pytest.mark.parametrize("name,tier", [("gpt1.3b", gs.OPT_STREAM), ("gpt1.3b", gs.OPT_HOST),
                                       ("gpt13b", gs.OPT_STREAM), ("gpt65b", gs.OPT_HOST)])
def test_bf16_production_path_matches_fp32_reference(name, tier):
    r = run_both(GEOMS[name], lp=2, alpha=ALPHA[name], opt_tier=tier)
    t = r["torch_amp"]
    bound = lambda k, floor: max(floor, 1.5 * t[k])  # noqa: E731
    assert r["loss"] < 2e-3
    assert r["m"] < bound("m", 2e-2) and r["fm"] < bound("fm", 2e-2)
    assert r["v"] < bound("v", 4e-2) and r["fv"] < bound("fv", 4e-2)
    assert r["dw"] < bound("dw", 0.15) and r["dfixed"] < bound("dfixed", 0.15)


@pytest.mark.parametrize("tier", [gs.OPT_STREAM, gs.OPT_HOST])
def test_fp32_mode_at_gpt1_3b_layer_geometry_holds_north_star_tolerances(tier):
    r = run_both(GEOMS["gpt1.3b"], lp=4, opt_tier=tier)
    assert r["loss"] < 1e-3
    assert r["w"] < 1e-4 and r["fixed"] < 1e-4


def _rel_rows(a, b, base=None):
    """norm-relative distance of two [N][P] float32 stacks (optionally of
    their deltas from `base`), accumulated per layer in float64 so no
    full-size float64 temporaries are made."""
    num = den = 0.0
    for l in range(len(b)):
        x = np.asarray(a[l], np.float64)
        y = np.asarray(b[l], np.float64)
        if base is not None:
            z = np.asarray(base[l], np.float64)
            x, y = x - z, y - z
        num += float(np.sum((x - y) ** 2))
        den += float(np.sum(y * y))
    return (num / den) ** 0.5


def test_bench_configuration_matches_fp32_reference():
    """bench.py's own workload, whole (BASELINE configs[1]: GPT-1.3B, all 24
    layers, M=16 micro-batches of b=2, s=2048, vertical plan with alpha=0.2,
    split (1,1,1), optimizer state in pinned DRAM stepped by the host cores,
    bench's Adam hyper-parameters and seed), two iterations through the
    product executor in bf16, against the same two iterations of
    tests/torch_ref.py in fp32 and under torch autocast-bf16 on the same
    tokens.  Gates: loss 2e-3; moments and parameter deltas within 2x of
    autocast's own distance from fp32."""
    torch = need_gpu()
    adam = dict(lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)
    g = ob.Geometry(n_layers=24, hidden=2048, heads=16, seq=2048, mb_size=2, vocab=50304)
    M, iters = 16, 2
    model = gs.ModelSpec(g.n_layers, g.hidden, g.heads, g.seq, g.mb_size, 2, 4, 3, 1)
    plan = gs.build_vertical(model, M, gs.StorageSplit(1.0, 1.0, 1.0), 0.2)
    eng = gs.Engine(plan, model, g.vocab, gs.AdamConfig(**adam), seed=1234, nvme_dir="/tmp", opt_tier=gs.OPT_HOST,
                    ssd_ring_layers=8)
    l0, f0 = eng.read_params()
    toks = np.stack([tr.tokens(g.vocab, g.mb_size, g.seq, M, it) for it in range(iters)])
    rep = eng.run(toks)
    eng.flush()
    l1, f1 = eng.read_params()
    m, v = eng.read_moments()
    eng.close()
    assert np.array_equal(rep.ledger, gs.plan_traffic(plan)), "executed ledger != plan ledger"
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    ref = tr.train(g, adam, l0, f0, toks, device="cuda", dtype="float32")
    torch.cuda.empty_cache()
    ours = dict(loss=float(np.max(np.abs(np.array(rep.losses) - ref["losses"]) / ref["losses"])),
                m=_rel_rows(m, ref["m"]), v=_rel_rows(v, ref["v"]), dw=_rel_rows(l1, ref["layers"], l0),
                dfixed=rel(f1 - f0, ref["fixed"] - f0))
    del m, v, l1
    amp = tr.train(g, adam, l0, f0, toks, device="cuda", dtype="float32", autocast_bf16=True)
    torch.cuda.empty_cache()
    t = dict(loss=float(np.max(np.abs(amp["losses"] - ref["losses"]) / ref["losses"])),
             m=_rel_rows(amp["m"], ref["m"]), v=_rel_rows(amp["v"], ref["v"]),
             dw=_rel_rows(amp["layers"], ref["layers"], l0), dfixed=rel(amp["fixed"] - f0, ref["fixed"] - f0))
    print(f"\nbench config (24 layers, M=16): losses {rep.losses} fp32 {ref['losses'].tolist()} "
          f"autocast {amp['losses'].tolist()} | ours " + " ".join(f"{k}={x:.3e}" for k, x in ours.items()) +
          " | torch autocast-bf16 " + " ".join(f"{k}={x:.3e}" for k, x in t.items()))
    # 2x autocast's distance here (1.5x for the 1-2 layer slices above): 24
    # layers of bf16 checkpoints, LN outputs and flash-style bf16 P / dS
    # compound; measured ours / autocast: m 2.0e-2 / 1.4e-2, v 1.7e-2 /
    # 1.2e-2, parameter deltas 9.7e-2 / 7.2e-2, loss 2.7e-6 / 5.2e-6
    # (profiles/round2/bench_config_parity_r4d.txt); a wrong gradient moves
    # these to O(1)
    bound = lambda k, floor: max(floor, 2.0 * t[k])  # noqa: E731
    assert ours["loss"] < 2e-3
    assert ours["m"] < bound("m", 2e-2)
    assert ours["v"] < bound("v", 4e-2)
    assert ours["dw"] < bound("dw", 0.15) and ours["dfixed"] < bound("dfixed", 0.15)
