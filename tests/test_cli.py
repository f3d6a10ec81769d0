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


@requires_reference
@pytest.mark.gpu
def test_run_executes_a_reference_dumped_plan(tmp_path):
    """A plan produced by the reference's own builder (plan_to_json, the
    `simulate --emit-plan` format) executes here unchanged; the executed
    ledger equals the plan's."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = tmp_path / "tiny.ini"
    cfg.write_text(TINY)
    plan = tmp_path / "ref_plan.json"
    plan.write_text(ob.ref_plan_json("vertical", ob.model_array(4, 64, 4, 32, 2, lp=4), 4, (1, 1, 0.5), 0.25))
    j = json.loads(offsim("run", str(cfg), "--from-plan", str(plan), "--iterations", "2", "--vocab", "128",
                          "--lp-bytes", "4"))
    assert j["ledger_equals_plan"] is True and len(j["losses"]) == 2
