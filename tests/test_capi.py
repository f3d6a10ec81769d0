"""The C-ABI library loads and exports every symbol include/greedysnake.h
declares (no GPU needed: no compute calls)."""
import ctypes as C
import os
import re

import paper_2512_17570_b200 as gs

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "greedysnake.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("gs_plan_build_vertical", "gs_engine_create", "gs_engine_run", "gs_gemm", "gs_adam_step_packed",
                 "gs_attention_fwd", "gs_vertical_traffic", "gs_simulate_json"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = gs.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_error_channel():
    lib = gs.lib()
    assert b"sm_100a" in lib.gs_version()
    h = C.c_void_p()
    rc = lib.gs_plan_from_json(b"not json", C.byref(h))
    assert rc == gs.ERR_VALIDATION
    assert b"malformed" in lib.gs_last_error()


def test_product_library_does_not_link_the_oracle():
    so = open(gs.LIB_PATH, "rb").read()
    assert b"gso_train" not in so and b"liboracle" not in so and b"ref_plan_json" not in so


def test_context_rejects_a_missing_device():
    # no compute: device -1 never exists (CPU container or GPU box alike)
    try:
        gs.Context(-1)
    except gs.OffsimError as e:
        assert "no CUDA device" in str(e)
    else:
        raise AssertionError("gs_ctx_create(-1) succeeded")


def test_io_roofline_is_infinite_without_ssd_state():
    model = gs.ModelSpec(24, 2048, 16, 2048, 2, 2, 4, 3, 1)
    m = gs.MachineSpec(gpu_mem_bytes=180 << 30, cpu_usable_dram_bytes=1 << 40, pcie_h2d_bw=5e10, pcie_d2h_bw=5e10,
                       ssd_read_bw=2.5e9, ssd_write_bw=2.5e9, fwd_compute_time_per_layer_per_mb=4e-4,
                       bwd_compute_time_per_layer_per_mb=1.2e-3, cpu_step_throughput=1e10, fixed_overhead_time=0.0,
                       num_gpus=1, gpu_working_set_bytes=1 << 30, ssd_duplex=True)
    assert gs.io_roofline(model, m, 32, 1.0) == float("inf")
    finite = gs.io_roofline(model, m, 32, 0.0)
    # 14.5 GB of optimizer state read and written (duplex) per 32 samples
    assert abs(finite - 32 / (12 * 50331648 * 24 / 2.5e9)) / finite < 1e-6
