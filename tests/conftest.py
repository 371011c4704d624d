import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref/libxpir_ref.so not built")
    try:
        return oracle.Ref()
    except OSError as e:  # libsodium missing on this host
        pytest.skip(f"reference build not loadable: {e}")


@pytest.fixture(scope="session")
def xp():
    """The product package; on a GPU box its CUDA library MUST load (no fallback)."""
    import paper_2001_08250_b200 as xp

    xp.lib()
    return xp


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a host without a visible CUDA device")
    return torch
