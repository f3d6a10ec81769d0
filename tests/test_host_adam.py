"""The host-core Adam (OptTier::Host CpuStep, engine/host_adam.cpp) is
bit-identical to a plain restatement of the update on this machine's CPU —
its AVX-512 path where the CPU has one, the scalar loop otherwise (CPU test:
builds tests/cpp/host_adam_check.cpp against the built objects)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "build", "gs", "engine")


@pytest.mark.skipif(not os.path.exists(os.path.join(OBJ, "host_adam.o")), reason="library not built")
def test_host_adam_bit_identical(tmp_path):
    exe = tmp_path / "host_adam_check"
    csrc = os.path.join(ROOT, "paper_2512_17570_b200", "csrc")
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{csrc}/engine", f"-I{ROOT}/include",
           f"-I{csrc}/kernels", "-I/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "host_adam_check.cpp"),
           os.path.join(OBJ, "host_adam.o"), os.path.join(OBJ, "host_tiers.o"), "-L/usr/local/cuda/lib64", "-lcudart",
           "-lpthread", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "lp=2: 0 differing" in r.stdout and "lp=4: 0 differing" in r.stdout
