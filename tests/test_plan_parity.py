"""Plan / ledger / simulator parity of the drop-in library against the
reference's own offsim library (oracle/_ref/liboffsim_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile).

* plan_to_json dumps are byte-identical over the grid of
  proj/tests/test_schedule.cpp:31-60 (N x M x split x alpha) plus dp>1,
  fp32 widths and the BASELINE geometries;
* closed-form ledgers equal the reference's and the plan sums;
* simulate() reports are byte-identical (report_to_json dump).
"""
import itertools
import json

import numpy as np
import pytest

import oracle_bindings as ob
import paper_2512_17570_b200 as gs

SPLITS = [(0, 0, 0), (1, 1, 1), (0.3, 0.7, 0.5), (0.123, 0.01, 0.999), (1, 1, 0.5), (1, 0, 0)]
ALPHAS = [0.0, 0.25, 0.5, 1.0]


def spec(n, h=64, s=128, b=2, heads=4, lp=2, dp=1):
    return gs.ModelSpec(n, h, heads, s, b, lp, 4, 3, dp), ob.model_array(n, h, heads, s, b, lp=lp, dp=dp)


def ref_or_none(fn):
    try:
        return fn()
    except RuntimeError as e:
        return ("error", str(e).split(":")[0])


def mine_or_none(fn):
    try:
        return fn()
    except gs.InfeasibleError:
        return ("error", "reference rc=3")
    except gs.ValidationError:
        return ("error", "reference rc=2")


@pytest.mark.parametrize("n,m", list(itertools.product([1, 2, 3, 4, 8], [1, 2, 3, 4, 8])))
def test_vertical_plans_byte_identical(n, m):
    mine_spec, ref_spec = spec(n)
    compared = 0
    for sp, a in itertools.product(SPLITS, ALPHAS):
        ref = ref_or_none(lambda: ob.ref_plan_json("vertical", ref_spec, m, sp, a))
        mine = mine_or_none(lambda: gs.build_vertical(mine_spec, m, gs.StorageSplit(*sp), a).to_json())
        assert ref == mine, (n, m, sp, a)
        compared += isinstance(mine, str)
    assert compared > 0


@pytest.mark.parametrize("n,m", list(itertools.product([1, 2, 4, 8], [1, 3, 8])))
def test_horizontal_plans_byte_identical(n, m):
    mine_spec, ref_spec = spec(n)
    for sp in SPLITS:
        ref = ob.ref_plan_json("horizontal", ref_spec, m, sp)
        mine = gs.build_horizontal(mine_spec, m, gs.StorageSplit(*sp)).to_json()
        assert ref == mine


@pytest.mark.parametrize("dp,lp", [(2, 2), (3, 2), (8, 2), (1, 4), (4, 4)])
def test_sharded_and_fp32_plans(dp, lp):
    mine_spec, ref_spec = spec(3, h=64, s=512, lp=lp, dp=dp)
    for sp, a, m in itertools.product(SPLITS, [0.0, 0.2], [1, 4]):
        ref = ref_or_none(lambda: ob.ref_plan_json("vertical", ref_spec, m, sp, a))
        mine = mine_or_none(lambda: gs.build_vertical(mine_spec, m, gs.StorageSplit(*sp), a).to_json())
        assert ref == mine


# BASELINE.json configs 2-5 geometries (ledger only: plans are large)
BASELINE = [
    ("1.3B", dict(n=24, h=2048, heads=16, s=2048, b=2), 16, (1, 1, 1), 0.0),
    ("13B", dict(n=40, h=5120, heads=40, s=2048, b=2), 32, (1, 1, 0), 0.2),
    ("65B", dict(n=80, h=8192, heads=64, s=2048, b=2), 32, (1, 1, 0.5), 0.2),
    ("65B-ssd", dict(n=80, h=8192, heads=64, s=2048, b=2), 32, (0, 0, 0), 0.0),
    ("175B", dict(n=96, h=12288, heads=96, s=2048, b=1), 32, (1, 0, 0), 0.2),
]


@pytest.mark.parametrize("name,geo,m,sp,a", BASELINE)
def test_baseline_ledgers_match_reference(name, geo, m, sp, a):
    for dp in (1, 2, 8):
        mine_spec, ref_spec = spec(geo["n"], geo["h"], geo["s"], geo["b"], geo["heads"], dp=dp)
        ref = ob.ref_ledger("vertical", ref_spec, m, sp, a)
        mine = gs.vertical_traffic(mine_spec, m, gs.StorageSplit(*sp), a)
        assert np.array_equal(ref, mine)
        ref_h = ob.ref_ledger("horizontal", ref_spec, m, sp)
        assert np.array_equal(ref_h, gs.horizontal_traffic(mine_spec, m, gs.StorageSplit(*sp)))


def test_1p3b_plan_sums_to_ledger_and_matches_reference():
    mine_spec, ref_spec = spec(24, 2048, 2048, 2, 16)
    plan = gs.build_vertical(mine_spec, 16, gs.StorageSplit(1, 1, 1), 0.2)
    assert plan.to_json() == ob.ref_plan_json("vertical", ref_spec, 16, (1, 1, 1), 0.2)
    assert np.array_equal(gs.plan_traffic(plan), gs.vertical_traffic(mine_spec, 16, gs.StorageSplit(1, 1, 1), 0.2))


def test_tiny_golden_ledger():
    """SURVEY.md §8(a) golden tiny ledger (M=4, split 0, alpha=0)."""
    mine_spec, _ = spec(4, 64, 32, 2)
    led = gs.vertical_traffic(mine_spec, 4, gs.StorageSplit(0, 0, 0), 0.0)
    want = np.array([[786432, 172032, 0, 73728, 0], [0, 131072, 786432, 73728, 0],
                     [786432, 98304, 0, 0, 2359296], [393216, 131072, 0, 0, 2359296]], np.uint64)
    assert np.array_equal(led, want)


MACHINE = [1 << 40, 1 << 44, 2.0e8, 1.5e8, 5.0e7, 4.0e7, 0.010, 0.021, 2.0e8, 0.0, 1, 1 << 20, 1]


@pytest.mark.parametrize("sp,a,duplex", [((0.5, 0.5, 0.5), 0.25, 1), ((1, 1, 0), 0.0, 0), ((0, 0, 0), 0.0, 1)])
def test_simulate_reports_byte_identical(sp, a, duplex):
    mine_spec, ref_spec = spec(4, 64, 128)
    plan = gs.build_vertical(mine_spec, 3, gs.StorageSplit(*sp), a)
    machine = list(MACHINE)
    machine[12] = duplex
    ref = ob.ref_simulate_json(plan.to_json(), machine)
    mine = gs.simulate(plan, gs.MachineSpec(*[int(x) if i in (0, 1, 10, 11) else x for i, x in enumerate(machine)]))
    assert json.loads(ref) == mine
    assert ref == json.dumps(mine, separators=(",", ":"))


def test_plan_json_round_trip():
    mine_spec, _ = spec(4, 64, 128)
    plan = gs.build_vertical(mine_spec, 3, gs.StorageSplit(0.5, 0.5, 0.5), 0.25)
    again = gs.SchedulePlan.from_json(plan.to_json())
    assert again.to_json() == plan.to_json()


def test_error_codes_follow_reference_taxonomy():
    mine_spec, _ = spec(4)
    with pytest.raises(gs.ValidationError):
        gs.build_vertical(mine_spec, 0, gs.StorageSplit(0, 0, 0), 0.0)
    with pytest.raises(gs.InfeasibleError):
        gs.build_vertical(mine_spec, 2, gs.StorageSplit(0, 0, 0), 0.5)
    with pytest.raises(gs.ValidationError):
        gs.SchedulePlan.from_json("{}")
