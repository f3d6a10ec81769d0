"""bench.py's driver contract on CPU: the reference arm's JSON line (the
oracle port timed on the host cores, `--impl reference`), the config block
naming the workload / optimizer tier / staging ring, and the rank-count
guard (a `--gpus N` run must not silently report a single rank)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("tiny:")


def test_config_names_tier_ring_and_batch():
    import argparse
    a = argparse.Namespace(config="gpt1.3b", microbatches=0, alpha=-1.0, schedule="vertical", gpus=1, ssd_ring=0,
                           opt_tier=-1)
    c = bench.config_dict(a)
    assert c["opt_tier"] == bench.OPT_TIERS[3] and "stepped by the host cores" in c["workload"]
    assert c["global_batch"] == 16 * 2 and c["seq_len"] == 2048 and c["split"] == [1.0, 1.0, 1.0]
    a.gpus, a.ssd_ring, a.opt_tier, a.microbatches = 8, 4, 1, 32
    c = bench.config_dict(a)
    assert c["global_batch"] == 32 * 2 * 8 and c["parallelism"] == "zero3-dp8"
    assert c["ssd_ring_layers"] == 4 and c["opt_tier"] == bench.OPT_TIERS[1]


def test_gpus_flag_must_match_the_launched_ranks():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "tiny"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "WORLD_SIZE" in (r.stderr + r.stdout)


@pytest.mark.parametrize("name", sorted(bench.CONFIGS))
def test_every_config_builds_its_plan(name):
    import paper_2512_17570_b200 as gs
    N, h, H, s, b, V, M, split, alpha, tier, ring = bench.CONFIGS[name]
    model = gs.ModelSpec(N, h, H, s, b, 2, 4, 3, 1)
    plan = gs.build_vertical(model, M, gs.StorageSplit(*split), alpha)
    assert len(plan) > 0 and tier in bench.OPT_TIERS and ring >= 1
