import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


HAVE_REFERENCE = os.path.isdir("/root/reference/proj")
requires_reference = pytest.mark.skipif(not HAVE_REFERENCE, reason="/root/reference not mounted")
