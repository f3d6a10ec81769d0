"""Pin the numeric CPU oracle (oracle/gs_oracle.c) against the torch float64
golden vectors (tools/make_golden.py -> tests/golden/tiny_golden.npz), and
check schedule invariance: executing the reference's vertical plan (any alpha)
gives the same training trajectory as the plain loop."""
import numpy as np
import pytest

import oracle_bindings as ob

GOLD = np.load(ob.os.path.join(ob.ROOT, "tests", "golden", "tiny_golden.npz"))
ADAM = dict(zip(("lr", "beta1", "beta2", "eps", "weight_decay"), GOLD["adam"].tolist()))
M = int(GOLD["microbatches"])


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def test_init_and_data_match_golden_bit_exact():
    layers, fixed = ob.init_params(ob.TINY)
    assert np.array_equal(layers, GOLD["init_layers"])
    assert np.array_equal(fixed, GOLD["init_fixed"])
    assert np.array_equal(ob.make_tokens(ob.TINY, int(GOLD["iters"]), M), GOLD["tokens"])


@pytest.mark.parametrize("split,alpha", [(None, None), ((0, 0, 0), 0.0), ((1, 1, 0), 0.25),
                                         ((1, 1, 1), 0.5), ((1, 1, 0.5), 1.0)])
def test_oracle_matches_torch_fp64(split, alpha):
    layers, fixed = ob.init_params(ob.TINY)
    plan = None if split is None else ob.ref_vertical_plan(ob.TINY, M, split, alpha)
    losses, p, f, _, _ = ob.train(ob.TINY, ADAM, M, plan, GOLD["tokens"], layers, fixed)
    # north-star tolerances: loss 1e-3 relative, params 1e-4 relative (norm-wise)
    assert np.max(np.abs(losses - GOLD["losses"]) / GOLD["losses"]) < 1e-5
    assert rel(p, GOLD["final_layers"]) < 1e-4
    assert rel(f, GOLD["final_fixed"]) < 1e-4


def test_delayed_step_without_flush_leaves_alpha_slice_stale():
    layers, fixed = ob.init_params(ob.TINY)
    plan = ob.ref_vertical_plan(ob.TINY, M, (1, 1, 1), 0.5)
    _, p_flush, _, _, _ = ob.train(ob.TINY, ADAM, M, plan, GOLD["tokens"], layers, fixed, flush=True)
    _, p_stale, _, _, _ = ob.train(ob.TINY, ADAM, M, plan, GOLD["tokens"], layers, fixed, flush=False)
    P = ob.TINY.P
    late = P - P // 2  # delayed slice = the last scaled_portion(P, alpha) elements
    assert np.array_equal(p_flush[:, :P - late], p_stale[:, :P - late])
    assert not np.array_equal(p_flush[:, P - late:], p_stale[:, P - late:])
