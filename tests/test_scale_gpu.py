"""Parity at the BASELINE configs' real sizes (BASELINE.json configs[1..4]).

Goldens (tests/golden/scale_*.npz) were made by oracle/gen_golden_scale.py
running the REFERENCE package itself: dense_reference (validate.py:83-111) on
the QFT-27 random input and on random 20q/24q x 20 circuits, and
min_sdrp_search (validate.py:280-300) on 54q x 7 circuits.  Each golden
keeps the reference output at 4096 seeded indices, 256 contiguous chunk
sums (a linear checksum of every amplitude) and the squared norm; the
inputs are regenerated bit-identically from their seeds.

Tolerances (north_star): per element 1e-12 (c128) / 1e-5 (c64).  Chunk sums
add 2^(n-8) elements, so they carry sqrt(2^(n-8)) x that.  QFT-34 has no CPU
oracle (256 GiB complex128): it is checked against the closed forms of the
QFT of GHZ and of a basis state on >= 4096 indices.
"""
from __future__ import annotations

import gc
import math

import numpy as np
import pytest

from paper_2304_14969_b200.circuit import Circuit, build_ghz, build_qft, build_random_circuit, x as x_gate
from paper_2304_14969_b200.executor import compile_circuit, dense_reference
from paper_2304_14969_b200.ket import DenseKet

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 1e-5}


def _random_state(width: int, seed: int) -> np.ndarray:
    """gen_golden_scale.random_state: the reference conftest.py:8-10 draw."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << width) + 1j * rng.normal(size=1 << width)
    v /= np.linalg.norm(v)
    return v


def _check_witnesses(y: np.ndarray, g, key: str, dtype: str, n: int) -> None:
    tol = TOL[dtype]
    idx = g[f"{key}/idx"]
    err = np.max(np.abs(y[idx] - g[f"{key}/amp"]))
    assert err < tol, f"{key} {dtype}: sampled max err {err:.3e}"
    chunk = y.reshape(256, -1).sum(axis=1)
    cerr = np.max(np.abs(chunk - g[f"{key}/chunk"]))
    assert cerr < tol * math.sqrt(1 << (n - 8)) * 4, f"{key} {dtype}: chunk-sum err {cerr:.3e}"
    nerr = abs(float(np.vdot(y, y).real) - float(g[f"{key}/norm2"]))
    assert nerr < (1e-10 if dtype == "c128" else 1e-5), f"{key} {dtype}: norm err {nerr:.3e}"


@pytest.fixture(scope="module")
def qft27(golden):
    g = golden("scale_qft27")
    n, seed = (int(v) for v in g["qft27/spec"])
    x = _random_state(n, seed)
    fft = np.fft.ifft(x) * math.sqrt(x.size)  # positive-exponent unitary DFT, every element
    return g, n, x, fft


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_qft27_random_input_vs_reference(qft27, dtype):
    """BASELINE configs[1]: the bench's own workload (random normalised input)
    through the drop-in API, checked against the reference's output on 4096
    indices + chunk sums, and against the DFT on every one of the 2^27 outputs."""
    g, n, x, fft = qft27
    assert float(g["qft27/fft_maxdiff"]) < 1e-12  # the golden itself agrees with the DFT
    y = dense_reference(build_qft(n), initial=DenseKet(n, x, dtype=dtype)).amps
    _check_witnesses(y, g, "qft27", dtype, n)
    err = float(np.max(np.abs(y - fft)))
    assert err < TOL[dtype], f"QFT-27 {dtype}: max |y - DFT(x)| = {err:.3e}"
    del y
    gc.collect()


@pytest.mark.parametrize("width", [20, 24])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_random_circuit_x20_vs_reference(golden, width, dtype):
    """BASELINE configs[2] family (Sycamore-style layers, depth 20) at the
    widths the reference itself can run (24q: 161 s on one core)."""
    g = golden(f"scale_rand{width}")
    key = f"rand{width}"
    w, depth, seed = (int(v) for v in g[f"{key}/spec"])
    y = dense_reference(build_random_circuit(w, depth, seed), dtype=dtype).amps
    _check_witnesses(y, g, key, dtype, w)


def _label_to_phys(order, labels: np.ndarray) -> np.ndarray:
    """Physical index of each label-order index when the readout permutation
    would be permute_qubits(state, order) (new bit k = old bit order[k])."""
    phys = np.zeros_like(labels)
    for k, o in enumerate(order):
        phys |= ((labels >> k) & 1) << o
    return phys


def _sampled(state: DenseKet, order, labels: np.ndarray) -> np.ndarray:
    phys = _label_to_phys(order, labels)
    return np.array([state.amplitude(int(i)) for i in phys])


def test_qft34_closed_forms_c64():
    """BASELINE configs[3] at 1 GPU: QFT-34 on a 128 GiB c64 state.  GHZ input:
    y_j = (1 + e^{-2 pi i j/N})/sqrt(2N); basis input |k>: y_j = e^{2 pi i jk/N}/sqrt(N);
    4096 random indices + index 0 and N-1 each."""
    n = 34
    N = 1 << n
    rng = np.random.default_rng(34)
    labels = np.unique(np.concatenate([rng.integers(0, N, 4096, dtype=np.int64), [0, N - 1]]))
    qft = compile_circuit(build_qft(n), dtype="c64")

    s = DenseKet(n, dtype="c64")
    compile_circuit(build_ghz(n), dtype="c64").run(s)
    qft.run(s)
    got = _sampled(s, qft.plan.order, labels)
    j = labels.astype(np.float64)
    want = (1.0 + np.exp(-2j * np.pi * j / N)) / math.sqrt(2.0 * N)
    err = np.max(np.abs(got - want))
    # amplitudes are ~1/sqrt(N) = 7.6e-6, so the absolute fp32 bound 1e-5 would be vacuous: 1e-4 relative
    assert err < 1e-4 / math.sqrt(N), f"QFT-34 GHZ: max err {err:.3e}"
    assert abs(s.norm() - 1.0) < 1e-4
    del s
    gc.collect()

    k = 0x2_5A5A_C3C3 & (N - 1)
    s = DenseKet(n, dtype="c64")
    compile_circuit(Circuit(n, tuple(x_gate(q) for q in range(n) if (k >> q) & 1)), dtype="c64").run(s)
    qft.run(s)
    got = _sampled(s, qft.plan.order, labels)
    want = np.exp(2j * np.pi * ((labels * k) % N).astype(np.float64) / N) / math.sqrt(N)
    err = np.max(np.abs(got - want))
    assert err < 1e-4 / math.sqrt(N), f"QFT-34 |k>: max err {err:.3e}"
    del s
    gc.collect()


STATS = ("label_swaps", "kernels", "eliminated_controls", "merges", "splits")


def _sdrp_cases(g):
    return sorted({k.rsplit("/", 1)[0] for k in g.files if k.startswith("sdrp54/")})


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_sdrp54_decisions_vs_reference(golden, dtype):
    """BASELINE configs[4]: 54q x 7 min-SDRP search (validate.py:280-300) on
    circuits derive_seed(0, 0..3) at 2^20 and 2^22 budgets: identical p_min and
    peak_amplitudes, F_model and every recorded eps of the p_min run within
    1e-9 (c128) / 1e-5 relative (c64)."""
    from paper_2304_14969_b200.engine import EngineConfig
    from paper_2304_14969_b200.sdrp import min_sdrp_search, run_hybrid

    g = golden("scale_sdrp54")
    for key in _sdrp_cases(g):
        w, depth, seed, budget = (int(v) for v in g[f"{key}/spec"])
        feasible, p_min, f_model, peak = g[f"{key}/res"]
        r = min_sdrp_search(w, depth, seed, budget, dtype=dtype)
        assert r.feasible == bool(feasible), key
        if not r.feasible:
            continue
        assert abs(r.p_min - p_min) < 1e-12, (key, dtype, r.p_min, p_min)
        assert r.peak_amplitudes == int(peak), (key, dtype)
        rel = 1e-9 if dtype == "c128" else 1e-4
        assert abs(r.f_model - f_model) <= rel * abs(f_model), (key, dtype, r.f_model, f_model)
        sim = run_hybrid(build_random_circuit(w, depth, seed),
                         EngineConfig(sdrp=p_min, mem_budget=budget, rng_seed=seed, dtype=dtype))
        sim.flush_all()
        want = g[f"{key}/eps"]
        assert len(sim.eps_record) == len(want), key
        np.testing.assert_allclose(sim.eps_record, want, atol=1e-9 if dtype == "c128" else 1e-5, err_msg=key)
