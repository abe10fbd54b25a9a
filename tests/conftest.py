"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full-size oracle comparisons)")


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (test infrastructure, oracle/)."""
    from oracle import oracle as O
    if not O.ORACLE_SO.exists():
        O.build(ref=False)
    return O


@pytest.fixture(scope="session")
def ref(oracle):
    """The reference translation units (oracle/_ref); skipped when unavailable."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    oracle.ref()
    return oracle


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1812_07122_b200 as P
    from paper_1812_07122_b200 import _capi
    _capi.lib()  # fail loudly if the extension is missing
    return P
