"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree CUDA library;
everything else runs on CPU (oracle vs golden vectors, host logic, ABI load)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN_DIR = ROOT / "tests" / "golden"
NETS_DIR = GOLDEN_DIR / "nets"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN_DIR / "golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def net_paths():
    return {p.stem: p for p in sorted(NETS_DIR.glob("*.json"))}


def golden_group(golden, prefix):
    """Sub-dict of golden arrays under prefix/ (prefix stripped)."""
    n = len(prefix) + 1
    return {k[n:]: v for k, v in golden.items() if k.startswith(prefix + "/")}
