"""Test configuration.

-m "not gpu": oracle pinned to the compiled reference + golden fixtures, host
              logic, the C-ABI library's exports, multi-process (gloo) logic.
-m gpu:       parity of the sm_100a path (through the C-ABI) against the
              oracle / golden fixtures on a B200.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def oracle():
    """The CPU checker (test infrastructure only)."""
    from oracle import pyoracle as O
    if not os.path.exists(O.LIB_PATH):
        O.build(ref=False)
    return O


@pytest.fixture(scope="session")
def ref(oracle):
    """The unmodified reference compiled from /root/reference (oracle/_ref)."""
    if not oracle.ref_available():
        if not os.path.isdir(oracle.REF_SRC):
            pytest.skip("reference library not built and /root/reference absent")
        oracle.build(ref=True)
    return oracle


@pytest.fixture(scope="session")
def kc():
    """The product package; its library must exist (no fallback)."""
    import paper_2512_00233_b200 as K
    if not os.path.exists(K.library_path()):
        from paper_2512_00233_b200 import build
        build.build()
    K.load_library()
    return K


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available() and torch.cuda.get_device_capability(0)[0] == 10
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu(kc):
    if not _has_gpu():
        pytest.fail("gpu test run without an sm_100 device (the path has no CPU fallback)")
    return kc


def golden(name):
    import json
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        return json.load(f)
