"""The `offsim` command line (paper_2512_17570_b200/bin/offsim): the
reference CLI's end-to-end checks (proj/tests/cli_end_to_end.cmake:1-80 —
output shape, determinism, plan round trip, exit codes) against this repo's
binary, plus byte parity of `simulate` / `plan` output with the reference
library (oracle/_ref) and a GPU `run` of a tiny configuration."""
import json
import os
import subprocess

import pytest

from conftest import requires_reference
import oracle_bindings as ob

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2512_17570_b200", "bin", "offsim")
DEMO = os.path.join(ROOT, "tests", "golden", "gpt65b_demo.ini")
TINY = """[model]
num_layers = 4
hidden_dim = 64
num_heads = 4
seq_len = 32
microbatch_size = 2

[machine]
gpu_mem_bytes = 100000000000
cpu_usable_dram_bytes = 50000000000
pcie_h2d_bw = 50e9
pcie_d2h_bw = 50e9
ssd_read_bw = 3e9
ssd_write_bw = 3e9
fwd_compute_time_per_layer_per_mb = 0.0002
bwd_compute_time_per_layer_per_mb = 0.0006
cpu_step_throughput = 1e10

[schedule]
variant = vertical
microbatches = 4
alpha = 0.25
x_ckpt = 1
x_param = 1
x_opt = 0.5
"""


def offsim(*args, rc=0):
    r = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == rc, (args, r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    return r.stdout


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(BIN):
        pytest.skip("offsim CLI not built (make -C paper_2512_17570_b200/csrc)")


def test_simulate_report_shape_and_determinism():
    a = offsim("simulate", DEMO)
    for key in ('"throughput"', '"traffic"', '"bound_class"'):
        assert key in a
    assert a == offsim("simulate", DEMO)


def test_sweep_compare_traffic_alloc_outputs():
    sweep = offsim("sweep", DEMO, "--m-range", "1..4", "--format", "csv")
    assert sweep.startswith("M,batch,throughput") and sweep.count("\n") >= 5
    cmp_ = offsim("compare", DEMO, "--schedules", "horizontal", "vertical@0.2")
    assert "horizontal" in cmp_ and "vertical" in cmp_
    assert "data_kind,H2D,D2H,SSD_read,SSD_write" in offsim("traffic", DEMO, "--format", "csv")
    assert json.loads(offsim("alloc-plan", "--count", "3", "--size", "4404019200"))["total_granted"] > 0


def test_plan_reports_the_papers_configuration():
    j = json.loads(offsim("plan", DEMO, "--oracle"))
    for key in ("microbatches", "alpha", "x_ckpt"):
        assert key in j
    # the reference planner's answer on the bundled demo
    assert j["microbatches"] == 19 and j["alpha"] == 0.32 and j["throughput_estimate"] == 0.121873
    assert j["oracle_max_deviation"] <= 0.01


def test_emit_and_replay_plan(tmp_path):
    p = tmp_path / "plan.json"
    emitted = offsim("simulate", DEMO, "--emit-plan", str(p))
    assert p.exists()
    assert offsim("simulate", DEMO, "--from-plan", str(p)) == emitted


def test_exit_codes(tmp_path):
    bad = tmp_path / "bad.cfg"
    bad.write_text("[model]\nnum_layers = -3\n")
    offsim("simulate", str(bad), rc=2)
    offsim("simulate", DEMO, "--microbatches", "1", "--alpha", "0.2", "--split", "0,0,0", rc=3)
    offsim("frobnicate", DEMO, rc=2)


@requires_reference
def test_simulate_matches_reference_report(tmp_path):
    p = tmp_path / "plan.json"
    mine = offsim("simulate", DEMO, "--emit-plan", str(p))
    machine = [40000000000, 380000000000, 24e9, 24e9, 3.2e9, 3.0e9, 0.068, 0.137, 1e9, 0.2, 1, 12000000000, 1.0]
    ref = json.loads(ob.ref_simulate_json(p.read_text(), machine))
    assert json.loads(mine) == ref


@pytest.mark.gpu
def test_run_tiny_config_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = tmp_path / "tiny.ini"
    cfg.write_text(TINY)
    j = json.loads(offsim("run", str(cfg), "--iterations", "2", "--vocab", "128", "--lp-bytes", "4"))
    assert j["ledger_equals_plan"] is True and len(j["losses"]) == 2 and j["measured_iteration_time"] > 0


GOLDEN_PLANS = os.path.join(ROOT, "tests", "golden", "ref_plans")
# name -> INI overrides of TINY for `run` (model geometry / precision of the dump)
GOLDEN_RUNS = {
    "tiny_vertical_split1_1_05_a025": dict(lp=4),
    "tiny_vertical_allssd_a0": dict(lp=4),
    "tiny_horizontal_split1_1_05": dict(lp=4),
    "tiny_vertical_bf16_split1_1_1_a02": dict(lp=2),
}


def golden(name):
    with open(os.path.join(GOLDEN_PLANS, name + ".json")) as f:
        plan = f.read()
    with open(os.path.join(GOLDEN_PLANS, name + ".ledger.json")) as f:
        led = json.load(f)
    return plan, led


def ini_for(led):
    N, h, H, s, b, lp = led["model"]
    x = led["split"]
    return TINY.replace("num_layers = 4", f"num_layers = {N}").replace("hidden_dim = 64", f"hidden_dim = {h}") \
        .replace("num_heads = 4", f"num_heads = {H}").replace("seq_len = 32", f"seq_len = {s}") \
        .replace("microbatch_size = 2", f"microbatch_size = {b}") \
        .replace("variant = vertical", f"variant = {led['variant']}") \
        .replace("microbatches = 4", f"microbatches = {led['microbatches']}") \
        .replace("alpha = 0.25", f"alpha = {led['alpha']}") \
        .replace("x_ckpt = 1", f"x_ckpt = {x[0]}").replace("x_param = 1", f"x_param = {x[1]}") \
        .replace("x_opt = 0.5", f"x_opt = {x[2]}")


@pytest.mark.parametrize("name", sorted(GOLDEN_RUNS))
def test_reference_dumped_plans_equal_this_builder(name):
    """The committed reference dumps (tools/make_ref_plans.py, from
    oracle/_ref) are byte-identical to this library's plan_to_json of the same
    configuration, and their ledgers to plan_traffic."""
    import numpy as np
    import paper_2512_17570_b200 as gs
    text, led = golden(name)
    N, h, H, s, b, lp = led["model"]
    m = gs.ModelSpec(N, h, H, s, b, lp, 4, 3, 1)
    split = gs.StorageSplit(*led["split"])
    plan = (gs.build_vertical(m, led["microbatches"], split, led["alpha"]) if led["variant"] == "vertical"
            else gs.build_horizontal(m, led["microbatches"], split))
    assert plan.to_json() == text
    assert np.array_equal(gs.plan_traffic(gs.SchedulePlan.from_json(text)), np.array(led["ledger"]))


@requires_reference
@pytest.mark.parametrize("name", sorted(GOLDEN_RUNS))
def test_golden_plans_are_what_the_reference_dumps(name):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import make_ref_plans  # noqa: E402
    plan, led = make_ref_plans.dump(name)
    text, gled = golden(name)
    assert plan == text and led["ledger"] == gled["ledger"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLDEN_RUNS))
def test_run_executes_a_reference_dumped_plan(tmp_path, name):
    """A plan produced by the reference's own builder (plan_to_json, the
    `simulate --emit-plan` format; committed under tests/golden/ref_plans)
    executes here unchanged (proj/tests/cli_end_to_end.cmake:64-72): the
    executed ledger equals the reference's, and the emitted trace is the
    plan (byte-identical once the per-task records are dropped) with every
    task executed once per iteration, in plan order on each resource queue
    (the in-order discipline of proj/src/simulator.cpp:108-126)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    text, led = golden(name)
    cfg = tmp_path / "cfg.ini"
    cfg.write_text(ini_for(led))
    plan = tmp_path / "ref_plan.json"
    plan.write_text(text)
    trace = tmp_path / "trace.json"
    iters = 3
    j = json.loads(offsim("run", str(cfg), "--from-plan", str(plan), "--iterations", str(iters), "--vocab", "128",
                          "--lp-bytes", str(GOLDEN_RUNS[name]["lp"]), "--emit-trace", str(trace)))
    assert j["ledger_equals_plan"] is True and len(j["losses"]) == iters
    rows = {"param": 0, "ckpt": 1, "grad_accum": 2, "interlayer_grad": 3, "opt_state": 4}
    cols = {"H2D": 0, "D2H": 1, "SSD_read": 2, "SSD_write": 3}
    for kind, per_link in j["traffic"].items():
        for link, v in per_link.items():
            assert v == led["ledger"][cols[link]][rows[kind]], (kind, link)
    tj = json.loads(trace.read_text())
    ref = json.loads(text)
    stripped = [{k: v for k, v in t.items() if k != "trace"} for t in tj["tasks"]]
    assert stripped == ref["tasks"]
    assert {k: v for k, v in tj.items() if k != "tasks"} == {k: v for k, v in ref.items() if k != "tasks"}
    per_res = {}
    for t in tj["tasks"]:
        assert sorted(r["iteration"] for r in t["trace"]) == list(range(iters)), t["id"]
        for r in t["trace"]:
            assert r["end_ms"] >= r["start_ms"] >= 0.0
            per_res.setdefault((r["resource"], r["iteration"]), []).append((r["start_ms"], t["id"]))
    for (res, it), recs in per_res.items():
        # one dispatcher thread / one in-order stream per resource: start
        # times are monotone in plan order
        starts = [s for s, _ in sorted(recs, key=lambda r: r[1])]
        assert all(b >= a - 1e-3 for a, b in zip(starts, starts[1:])), (res, it)
