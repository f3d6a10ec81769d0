"""The reference's own unit suites (proj/tests/test_*.cpp, compiled in place
through tests/cpp/doctest.h) pass against this repo's drop-in offsim library
and against the reference library itself (sanity of the shim)."""
import os
import subprocess

import pytest

from conftest import requires_reference

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["test_model", "test_machine", "test_traffic", "test_schedule", "test_simulator", "test_roofline",
          "test_json_io", "test_simplex", "test_planner", "test_config", "test_alloc"]


@pytest.fixture(scope="module")
def built():
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "-j8"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return os.path.join(ROOT, "build", "conformance")


@requires_reference
@pytest.mark.parametrize("suite", SUITES)
@pytest.mark.parametrize("lib", ["gs", "ref"])
def test_reference_suite(built, suite, lib):
    r = subprocess.run([os.path.join(built, lib, suite)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout


@requires_reference
@pytest.mark.parametrize("lib", ["gs", "ref"])
def test_reference_acceptance_binary(built, lib):
    """The reference's acceptance criteria c1-c10 (proj/tests/acceptance.cpp:
    plan == ledger, memory caps, roofline containment, full-SSD plateau, the
    demo's vertical/horizontal ratio, ...) against this repo's library (gs)
    and the reference's own (ref)."""
    exe = os.path.join(built, "gs", "acceptance") if lib == "gs" else os.path.join(ROOT, "oracle", "_ref", "acceptance")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "all criteria passed" in r.stdout, r.stdout[-3000:]
    for c in range(1, 11):
        assert f"PASS criterion {c:2d}:" in r.stdout
