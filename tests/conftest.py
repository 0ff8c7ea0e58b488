"""Shared fixtures.

-m "not gpu": the CPU checkers (oracle/) against the reference's own golden
vectors and SPEC examples, host logic, and that the sm_100a library loads and
exports the C-ABI. -m gpu: device-vs-oracle parity through the C-ABI.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1610_07159_b200 import build as _build  # noqa: E402
from paper_1610_07159_b200.hwflow import Solver  # noqa: E402

GOLDEN = ROOT / "tests" / "golden" / "ref_small.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libhwflow_cuda.so")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    """The plain-C++ restatement (test infrastructure only)."""
    if not _build.ORACLE_LIB.exists():
        _build.build_oracle()
    return Solver(_build.ORACLE_LIB)


@pytest.fixture(scope="session")
def reference():
    """The reference's own sources compiled against the Eigen shim (skipped if not built)."""
    if not _build.REF_LIB.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Solver(_build.REF_LIB)


@pytest.fixture(scope="session")
def device():
    """The product: fails loudly (no skip) when the CUDA library or the GPU is missing."""
    if not _build.CUDA_LIB.exists():
        _build.build_cuda()
    s = Solver(_build.CUDA_LIB)
    assert s.backend == "cuda-sm_100a"
    return s
