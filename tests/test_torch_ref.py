"""Pins tests/torch_ref.py (the torch restatement the production-geometry GPU
parity tests compare against) to the committed torch-fp64 golden and to the
C oracle, on CPU at the tiny geometry (proj/tests/helpers.hpp:10-19)."""
import numpy as np
import pytest

import oracle_bindings as ob
import torch_ref as tr

GOLD = np.load(ob.os.path.join(ob.ROOT, "tests", "golden", "tiny_golden.npz"))
ADAM = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def test_init_and_tokens_match_oracle():
    g = ob.Geometry(n_layers=3, hidden=32, heads=2, seq=16, mb_size=2, vocab=97)
    l0, _ = ob.init_params(g)
    for l in range(g.n_layers):
        assert np.array_equal(tr.layer_init_at(g.n_layers, g.hidden, 42, l, np.arange(g.P)), l0[l])
    ref = ob.make_tokens(g, 3, 4)
    for it in range(3):
        assert np.array_equal(tr.tokens(g.vocab, g.mb_size, g.seq, 4, it), ref[it])


def test_fp64_restatement_reproduces_golden():
    pytest.importorskip("torch")
    g = ob.TINY
    out = tr.train(g, ADAM, GOLD["init_layers"], GOLD["init_fixed"], GOLD["tokens"], dtype="float64")
    assert np.max(np.abs(out["losses"] - GOLD["losses"]) / GOLD["losses"]) < 1e-12
    assert rel(out["layers"], GOLD["final_layers"]) < 1e-7
    assert rel(out["fixed"], GOLD["final_fixed"]) < 1e-7


def test_fp32_restatement_matches_c_oracle():
    pytest.importorskip("torch")
    g, M = ob.TINY, 4
    l0, f0 = ob.init_params(g)
    toks = ob.make_tokens(g, 3, M)
    out = tr.train(g, ADAM, l0, f0, toks, dtype="float32")
    losses, layers, fixed, (m, v), _ = ob.train(g, ADAM, M, None, toks, l0, f0)
    assert np.max(np.abs(out["losses"] - losses) / losses) < 1e-5
    assert rel(out["layers"], layers) < 1e-5
    assert rel(out["fixed"], fixed) < 1e-5
    assert rel(out["m"], m) < 1e-4 and rel(out["v"], v) < 1e-4
