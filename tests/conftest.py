"""Shared fixtures; registers the `gpu` marker (tests needing a B200)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the libshardcu kernels")


def random_state(width: int, rng) -> np.ndarray:
    """Seeded normalised complex Gaussian state (reference conftest.py:8-10)."""
    v = rng.normal(size=1 << width) + 1j * rng.normal(size=1 << width)
    return v / np.linalg.norm(v)


def random_unitary(rng) -> np.ndarray:
    """Haar-ish 2x2 unitary (reference conftest.py:13-16)."""
    z = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def naive_apply(amps, width, m, target, controls=(), polarity=()):
    """Index-by-index gate oracle sharing no code with any kernel
    (reference conftest.py:19-33)."""
    out = np.zeros_like(amps)
    for idx, amp in enumerate(amps):
        if any(((idx >> c) & 1) != pol for c, pol in zip(controls, polarity)):
            out[idx] += amp
            continue
        bit = (idx >> target) & 1
        out[idx & ~(1 << target)] += m[0, bit] * amp
        out[idx | (1 << target)] += m[1, bit] * amp
    return out


def reduced_density(amps, width, q):
    """Partial-trace oracle (reference conftest.py:55-62)."""
    rho = np.zeros((2, 2), dtype=complex)
    for i, ai in enumerate(amps):
        for b in (0, 1):
            j = (i & ~(1 << q)) | (b << q)
            rho[(i >> q) & 1, b] += ai * np.conj(amps[j])
    return rho


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    return load


def has_gpu() -> bool:
    try:
        from paper_2304_14969_b200 import _lib
        return _lib.device_count() > 0
    except Exception:
        return False
