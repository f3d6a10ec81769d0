"""Data parallelism through the product executor: two
ranks, each its own process and Engine (world = 2, ZeRO-3 shards), their
collectives over peer memory (engine/peer_comm.hpp: CUDA IPC mappings, stream
counters, the rank-ordered reduce kernel).  Both processes share cuda:0 when
the box has one GPU — the same IPC / counter protocol an 8-GPU NVSwitch node
runs, with HBM in place of NVLink.

Reference: single-process training on all W * M micro-batches (the oracle's
plain loop; the vertical plan with its alpha-delayed step equals it after
flush()).  Rank r runs global micro-batches
[r*M, (r+1)*M) of each iteration; the shard layout is shard_range.
Tolerances: the north star's fp32 gates (loss 1e-3, parameters 1e-4).
"""
import multiprocessing as mp
import os
import traceback

import numpy as np
import pytest

import oracle_bindings as ob

pytestmark = pytest.mark.gpu

ADAM = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)
G = ob.Geometry(n_layers=4, hidden=64, heads=4, seq=32, mb_size=2, vocab=128)
M, W, ITERS = 2, 2, 3


def worker(rank, comm_id, cfg, out):
    try:
        import paper_2512_17570_b200 as gs
        split, alpha, tier = cfg
        model = gs.ModelSpec(G.n_layers, G.hidden, G.heads, G.seq, G.mb_size, 4, 4, 3, W)
        plan = gs.build_vertical(model, M, gs.StorageSplit(*split), alpha)
        eng = gs.Engine(plan, model, G.vocab, gs.AdamConfig(**ADAM), seed=42, device=0, nvme_dir="/tmp",
                        opt_tier=tier, rank=rank, world=W, comm_id=comm_id)
        tokens = ob.make_tokens(G, ITERS, M * W)
        mine = np.ascontiguousarray(tokens[:, rank * M:(rank + 1) * M])
        rep = eng.run(mine)
        eng.flush()
        layers, fixed = eng.read_params()
        ledger = rep.ledger
        want = gs.plan_traffic(plan)
        eng.close()
        np.savez(out, losses=np.array(rep.losses), layers=layers, fixed=fixed, ledger_ok=np.array_equal(ledger, want),
                 launches=rep.gpu_launches)
    except Exception:  # surfaced by the parent
        with open(out + ".err", "w") as f:
            f.write(traceback.format_exc())


def run_world2(tmp_path, cfg):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2512_17570_b200 as gs
    comm_id = gs.comm_unique_id()
    ctx = mp.get_context("spawn")
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(W)]
    procs = [ctx.Process(target=worker, args=(r, comm_id, cfg, outs[r])) for r in range(W)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for p in procs:
        if p.is_alive():  # never leave a hung rank behind
            p.kill()
            p.join()
            pytest.fail("a data-parallel rank hung")
    for o in outs:
        if os.path.exists(o + ".err"):
            pytest.fail(open(o + ".err").read())
    return [np.load(o) for o in outs]


@pytest.mark.parametrize("cfg", [((1, 1, 0.5), 0.25, 0), ((1, 1, 1), 0.25, 3), ((0, 0, 0), 0.0, 2)],
                         ids=["nvme-half-hbm-opt", "dram-host-step", "all-ssd-stream"])
def test_world2_executor_matches_single_process_oracle(tmp_path, cfg):
    res = run_world2(tmp_path, cfg)
    layers0, fixed0 = ob.init_params(G)
    tokens = ob.make_tokens(G, ITERS, M * W)
    ref_loss, ref_layers, ref_fixed, _, _ = ob.train(G, ADAM, M * W, None, tokens, layers0, fixed0)
    # every rank's executed ledger is its plan's (per-GPU shard bytes)
    assert all(bool(r["ledger_ok"]) for r in res)
    # the global loss is the mean over the ranks' micro-batches
    loss = np.mean([r["losses"] for r in res], axis=0)
    assert np.max(np.abs(loss - ref_loss) / ref_loss) < 1e-3
    # ZeRO-3: each rank holds (and reports) its own shard of every layer
    P = G.P
    layers = np.zeros_like(ref_layers)
    for rank, r in enumerate(res):
        lo, hi = rank * (P // W), (rank + 1) * (P // W)
        layers[:, lo:hi] = r["layers"][:, lo:hi]
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    assert rel(layers, ref_layers) < 1e-4
    # the tied embedding is replicated: identical on both ranks, equal to the oracle's
    assert np.array_equal(res[0]["fixed"], res[1]["fixed"])
    assert rel(res[0]["fixed"], ref_fixed) < 1e-4


def _bench_line(args, timeout=900):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=root, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_contract_line_single_gpu():
    """bench.py's driver line on the GPU (tiny config): every contract key,
    the executed ledger equal to the plan's, kernels launched."""
    d = _bench_line(["--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--calibrate", "0"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0 and d["ledger_equals_plan"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k


def test_bench_two_ranks_through_torchrun():
    """`bench.py --gpus 2` re-launches itself under torch.distributed.run; the
    two ranks (sharing the box's GPU when it has one) run the ZeRO-3
    peer-memory path and rank 0 reports n_gpus 2."""
    d = _bench_line(["--gpus", "2", "--share-gpu", "--config", "tiny", "--steps", "2", "--warmup", "3",
                     "--no-cpu-baseline", "--calibrate", "0"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["ledger_equals_plan"]
    assert d["config"]["parallelism"] == "zero3-dp2" and d["config"]["global_batch"] == 2 * 4 * 2
