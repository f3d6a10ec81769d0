"""Planner parity: this repo's solve_config /
grid_search_config / find_optimal_config / solve_lp against the reference's
own planner (oracle/_ref/liboffsim_ref.so, proj/src/planner.cpp and
simplex.cpp compiled in place), on randomised machines in the style of
proj/tests/test_planner.cpp:13-42 plus the BASELINE geometries.

Floating-point tolerance: stage times and throughputs agree within 1e-9
relative (same model, independent LP implementation); splits within 1e-6
where the LP optimum is unique (regulariser + lexicographic nudge)."""
import random

import numpy as np
import pytest

from conftest import requires_reference
import oracle_bindings as ob
import paper_2512_17570_b200 as gs


def machine(rng):
    m = dict(gpu_mem_bytes=80 << 30, cpu_usable_dram_bytes=1 << rng.randint(22, 34), pcie_h2d_bw=rng.uniform(1e7, 1e10),
             pcie_d2h_bw=rng.uniform(1e7, 1e10), ssd_read_bw=rng.uniform(1e6, 1e9), ssd_write_bw=rng.uniform(1e6, 1e9),
             fwd_compute_time_per_layer_per_mb=rng.uniform(0.001, 0.3),
             bwd_compute_time_per_layer_per_mb=rng.uniform(0.001, 0.3), cpu_step_throughput=rng.uniform(1e7, 1e10),
             fixed_overhead_time=rng.uniform(0, 0.1), num_gpus=rng.choice([1, 2, 8]), gpu_working_set_bytes=1 << 28,
             ssd_duplex=rng.random() < 0.5)
    arr = [m["gpu_mem_bytes"], m["cpu_usable_dram_bytes"], m["pcie_h2d_bw"], m["pcie_d2h_bw"], m["ssd_read_bw"],
           m["ssd_write_bw"], m["fwd_compute_time_per_layer_per_mb"], m["bwd_compute_time_per_layer_per_mb"],
           m["cpu_step_throughput"], m["fixed_overhead_time"], m["num_gpus"], m["gpu_working_set_bytes"],
           1.0 if m["ssd_duplex"] else 0.0]
    return gs.MachineSpec(**m), arr


def close(a, b, rel=1e-9):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def same(mine: gs.PlannerSolution, ref, split_tol=1e-6):
    assert mine.feasible == bool(ref[0])
    if not mine.feasible:
        return
    assert mine.num_microbatches == int(ref[1]) and close(mine.alpha, ref[2])
    assert close(mine.t_fwd_stage + mine.t_bwd_stage, ref[6] + ref[7], 1e-6)
    assert close(mine.iteration_estimate, ref[8], 1e-6) and close(mine.throughput_estimate, ref[9], 1e-6)
    sp = (mine.split.x_ckpt, mine.split.x_param, mine.split.x_opt)
    assert np.allclose(sp, ref[3:6], atol=split_tol), (sp, ref[3:6])


@requires_reference
@pytest.mark.parametrize("seed", range(8))
def test_solve_config_matches_reference(seed):
    rng = random.Random(1000 + seed)
    for _ in range(12):
        n, h, mbs = rng.randint(2, 12), rng.choice([64, 128, 256]), rng.randint(1, 8)
        dp = rng.choice([1, 1, 2, 4])
        model = gs.ModelSpec(n, h, 4, 256, 2, 2, 4, 3, dp)
        ref_model = ob.model_array(n, h, 4, 256, 2, dp=dp)
        mc, arr = machine(rng)
        alpha = rng.uniform(0, 0.5)
        same(gs.solve_config(model, mc, mbs, alpha), ob.ref_planner("solve", ref_model, arr, mbs, alpha))


@requires_reference
@pytest.mark.parametrize("seed", range(3))
def test_grid_search_matches_reference(seed):
    rng = random.Random(77 + seed)
    for _ in range(3):
        n, mbs = rng.randint(2, 8), rng.randint(1, 6)
        model = gs.ModelSpec(n, 128, 4, 256, 2, 2, 4, 3, 1)
        mc, arr = machine(rng)
        alpha = rng.uniform(0, 0.5)
        mine = gs.grid_search_config(model, mc, mbs, alpha, 20)
        ref = ob.ref_planner("grid", ob.model_array(n, 128, 4, 256, 2), arr, mbs, alpha, 20)
        same(mine, ref, split_tol=1e-12)


@requires_reference
@pytest.mark.parametrize("geometry", [(24, 2048, 16, 2), (40, 5120, 40, 2), (80, 8192, 64, 2), (96, 12288, 96, 1)])
def test_find_optimal_config_matches_reference_at_baseline_geometries(geometry):
    """Algorithm 1 on the BASELINE models with a B200-box machine (measured
    PCIe / virtio-disk rates, engine per-layer times scaled by h^2)."""
    n, h, heads, b = geometry
    model = gs.ModelSpec(n, h, heads, 2048, b, 2, 4, 3, 1)
    scale = (h / 2048) ** 2 * b / 2
    mc = gs.MachineSpec(gpu_mem_bytes=180 << 30, cpu_usable_dram_bytes=190 << 30, pcie_h2d_bw=49e9, pcie_d2h_bw=49e9,
                        ssd_read_bw=2.6e9, ssd_write_bw=2.6e9, fwd_compute_time_per_layer_per_mb=0.43e-3 * scale,
                        bwd_compute_time_per_layer_per_mb=1.29e-3 * scale, cpu_step_throughput=16e9,
                        fixed_overhead_time=0.009, num_gpus=1, gpu_working_set_bytes=8 << 30, ssd_duplex=True)
    arr = [mc.gpu_mem_bytes, mc.cpu_usable_dram_bytes, mc.pcie_h2d_bw, mc.pcie_d2h_bw, mc.ssd_read_bw, mc.ssd_write_bw,
           mc.fwd_compute_time_per_layer_per_mb, mc.bwd_compute_time_per_layer_per_mb, mc.cpu_step_throughput,
           mc.fixed_overhead_time, 1, mc.gpu_working_set_bytes, 1.0]
    mine = gs.find_optimal_config(model, mc)
    ref = ob.ref_planner("optimal", ob.model_array(n, h, heads, 2048, b), arr)
    assert mine.feasible == bool(ref[0]) and mine.num_microbatches == int(ref[1])
    if not mine.feasible:  # 65B / 175B: the fp32 grads alone exceed this box's DRAM
        return
    assert close(mine.throughput_estimate, ref[9], 1e-9)
    # alphas whose projections tie to the last bits are interchangeable: the
    # reference's own planner must rate ours equal to its pick
    again = ob.ref_planner("solve", ob.model_array(n, h, heads, 2048, b), arr, mine.num_microbatches, mine.alpha)
    assert close(again[9], ref[9], 1e-9)


@requires_reference
def test_solve_lp_matches_reference():
    rng = random.Random(5)
    for _ in range(200):
        m, n = rng.randint(1, 8), rng.randint(1, 5)
        A = [[rng.uniform(-3, 3) for _ in range(n)] for _ in range(m)]
        b = [rng.uniform(-2, 6) for _ in range(m)]
        c = [rng.uniform(-2, 2) for _ in range(n)]
        f, bd, obj, x = gs.solve_lp(A, b, c)
        rf, rbd, robj, rx = ob.ref_solve_lp(A, b, c)
        assert f == rf
        if f:
            assert bd == rbd
            if bd:
                assert abs(obj - robj) <= 1e-7 * max(1.0, abs(robj))
                for i in range(m):
                    assert sum(A[i][j] * x[j] for j in range(n)) <= b[i] + 1e-7
                assert min(x) >= -1e-9


@requires_reference
@pytest.mark.parametrize("seed", range(20))
def test_rooflines_match_reference(seed):
    """io_roofline / compute_roofline (roofline.cpp:8-33) through the C-ABI."""
    rng = random.Random(1000 + seed)
    m, arr = machine(rng)
    n, h, dp = rng.randint(2, 96), rng.choice([64, 2048, 8192]), rng.choice([1, 2, 8])
    model = gs.ModelSpec(n, h, 4, 256, 2, 2, 4, 3, dp)
    x_opt = rng.choice([0.0, 0.25, 0.5, 1.0])
    batch = rng.choice([1, 4, 64])
    io_ref, comp_ref = ob.ref_rooflines(ob.model_array(n, h, 4, 256, 2, dp=dp), arr, batch, x_opt)
    io = gs.io_roofline(model, m, batch, x_opt)
    comp = gs.compute_roofline(model, m)
    assert (io == io_ref == float("inf")) or close(io, io_ref)
    assert close(comp, comp_ref)
