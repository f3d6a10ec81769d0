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
