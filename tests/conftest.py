"""Shared pytest configuration.

Markers: ``gpu`` — needs a CUDA device (B200); these are the parity tests proper
and go through the C ABI (librcp_b200.so).  Everything else runs on CPU.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librcp_b200.so")
    config.addinivalue_line("markers", "slow: long-running (large n)")


def golden_names():
    """Small reference fixtures (inputs stored or cheap to regenerate); the full-size
    BASELINE fixtures g_full_* are read by tests/test_full_size.py only."""
    return sorted(p.stem for p in GOLDEN.glob("g_*.npz") if not p.stem.startswith("g_full_"))


def load_golden(name):
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["cfg"] = json.loads(str(d["cfg"]))
    d["spec"] = json.loads(str(d["spec"]))
    d["robust"] = bool(d["robust"])
    if "a" not in d:
        from paper_1710_00125_b200 import gallery
        sp = d["spec"]
        d["a"] = gallery.type6(sp["n"], sp["seed"])
    return d


def l_tol(n: int) -> float:
    """Stated L/D parity tolerance (absolute on L, relative to max|D| on D).

    10x the CPU-vs-perturbed-CPU noise floor measured in SURVEY.md section 7.3
    (max|dL| ~ 7e-14 at n=256, 5e-13 at n=1000, 3.6e-12 at n=4096, ~ n^1.5).
    """
    return max(1e-12, 3e-15 * n ** 1.5)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a CUDA device"
    from paper_1710_00125_b200 import _native
    _native.load()  # raises NativeUnavailable: no fallback
    return True
