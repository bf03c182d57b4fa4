"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference's dense ket hot path
(/root/reference/pkg/src/shardsim/ket.py and the dense loop of
validate.py:83-111), complex128, single-threaded, kernel-identical
arithmetic (the same view-based NumPy expressions per kernel).

Who may use it: tests/ (as the checker), __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference leg (as the timed
reference CPU path).  The product (paper_2304_14969_b200) never imports it.

Parity of this oracle is PINNED: tests/test_oracle_golden.py checks every
function against tests/golden/*.npz, which oracle/gen_golden.py produced by
importing and running the reference package itself.
"""
from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# views (ket.py:99-122)
# ---------------------------------------------------------------------------


def _views(amps: np.ndarray, width: int, q: int, controls=(), polarity=()):
    """(bit-0 view, bit-1 view) of qubit q restricted to matching controls."""
    t = amps.reshape((2,) * width)
    sel = [slice(None)] * width
    for c, pol in zip(controls, polarity):
        a = width - 1 - c
        sel[a] = slice(pol, pol + 1)
    axis = width - 1 - q
    s0, s1 = list(sel), list(sel)
    s0[axis] = slice(0, 1)
    s1[axis] = slice(1, 2)
    return t[tuple(s0)], t[tuple(s1)]


def _width(amps: np.ndarray) -> int:
    return int(amps.size).bit_length() - 1


# ---------------------------------------------------------------------------
# kernels (ket.py:128-233)
# ---------------------------------------------------------------------------


def apply_1q(amps: np.ndarray, q: int, m: np.ndarray) -> None:
    """In place; ket.py:133-144 (diagonal fast path :136-138)."""
    a0, a1 = _views(amps, _width(amps), q)
    if abs(m[0, 1]) == 0.0 and abs(m[1, 0]) == 0.0:
        a0 *= m[0, 0]
        a1 *= m[1, 1]
    else:
        new0 = m[0, 0] * a0 + m[0, 1] * a1
        a1 *= m[1, 1]
        a1 += m[1, 0] * a0
        a0[...] = new0


def apply_controlled(amps: np.ndarray, controls, polarity, target: int, m: np.ndarray) -> None:
    """In place; ket.py:146-164 (identity entries skipped :154-158)."""
    a0, a1 = _views(amps, _width(amps), target, controls, polarity)
    if abs(m[0, 1]) == 0.0 and abs(m[1, 0]) == 0.0:
        if m[0, 0] != 1.0:
            a0 *= m[0, 0]
        if m[1, 1] != 1.0:
            a1 *= m[1, 1]
    else:
        new0 = m[0, 0] * a0 + m[0, 1] * a1
        a1 *= m[1, 1]
        a1 += m[1, 0] * a0
        a0[...] = new0


def apply_pauli_layer(amps: np.ndarray, ops) -> np.ndarray:
    """Returns the new array; ket.py:166-202 (phase belongs to the source)."""
    flip = sign = y = 0
    for q, p in ops:
        if p == "x":
            flip |= 1 << q
        elif p == "y":
            flip |= 1 << q
            sign |= 1 << q
            y += 1
        elif p == "z":
            sign |= 1 << q
        else:
            raise ValueError(p)
    n = amps.size
    scale = 1j ** (y % 4)
    if sign:
        idx = np.arange(n, dtype=np.uint64)
        parity = np.bitwise_count(idx & np.uint64(sign)) & np.uint64(1)
        phases = np.where(parity.astype(bool), -scale, scale)
    else:
        phases = scale
    if flip:
        src = np.arange(n, dtype=np.intp) ^ flip
        return amps[src] * (phases[src] if sign else phases)
    return amps * phases


def bloch_sums(amps: np.ndarray, q: int):
    """(Re, Im of sum conj(a0) a1, sum |a0|^2, sum |a1|^2); ket.py:204-210."""
    a0, a1 = _views(amps, _width(amps), q)
    cross = np.sum(np.conj(a0) * a1)
    return (float(cross.real), float(cross.imag), float(np.sum(np.abs(a0) ** 2)),
            float(np.sum(np.abs(a1) ** 2)))


def bloch_vector(amps: np.ndarray, q: int):
    cr, ci, n0, n1 = bloch_sums(amps, q)
    return (2.0 * cr, 2.0 * ci, n0 - n1)


def epsilon(r) -> float:
    """ket.py:37-39."""
    return (1.0 - min(math.sqrt(r[0] ** 2 + r[1] ** 2 + r[2] ** 2), 1.0)) / 2.0


def probability(amps: np.ndarray, q: int, outcome: int) -> float:
    a0, a1 = _views(amps, _width(amps), q)
    return float(np.sum(np.abs(a0 if outcome == 0 else a1) ** 2))


def project_and_renormalize(amps: np.ndarray, q: int, outcome: int) -> float:
    """In place; ket.py:212-226."""
    a0, a1 = _views(amps, _width(amps), q)
    keep, drop = (a0, a1) if outcome == 0 else (a1, a0)
    prob = float(np.sum(np.abs(keep) ** 2))
    if prob <= 1e-12:
        raise ValueError(f"outcome {outcome} on qubit {q} has probability {prob:.3e}")
    drop[...] = 0.0
    keep *= 1.0 / math.sqrt(prob)
    return prob


def kron_compose(lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """ket.py:239-241: `lo` keeps the low positions."""
    return np.kron(hi, lo)


def try_decompose(amps: np.ndarray, q: int, tol: float):
    """ket.py:243-267; returns (phi[2], rest) or None."""
    w = _width(amps)
    if w < 2:
        return None
    if epsilon(bloch_vector(amps, q)) > tol:
        return None
    a0, a1 = _views(amps, w, q)
    p0 = float(np.sum(np.abs(a0) ** 2))
    dominant = a0 if p0 >= 0.5 else a1
    rest = (dominant / math.sqrt(max(p0, 1.0 - p0))).reshape(-1)
    phi = np.array([np.vdot(rest, a0.reshape(-1)), np.vdot(rest, a1.reshape(-1))])
    phi /= np.sqrt(np.sum(np.abs(phi) ** 2))
    rest = rest / np.sqrt(np.sum(np.abs(rest) ** 2))
    return phi, rest


def remove_qubit(amps: np.ndarray, q: int) -> np.ndarray:
    """ket.py:269-275."""
    a0, a1 = _views(amps, _width(amps), q)
    residual = float(np.sum(np.abs(a1) ** 2))
    if residual > 1e-9:
        raise ValueError(f"qubit {q} is not in |0> (residual {residual:.3e})")
    return a0.reshape(-1).copy()


def fidelity(a: np.ndarray, b: np.ndarray) -> float:
    """ket.py:277-281."""
    return float(np.abs(np.vdot(a, b)) ** 2)


def permute_qubits(amps: np.ndarray, order) -> np.ndarray:
    """ket.py:284-292: new qubit k is old qubit order[k]."""
    w = _width(amps)
    axes = [w - 1 - order[w - 1 - a] for a in range(w)]
    return np.transpose(amps.reshape((2,) * w), axes).reshape(-1).copy()


def bloch_to_state(r) -> np.ndarray:
    """ket.py:42-54."""
    norm = math.sqrt(r[0] ** 2 + r[1] ** 2 + r[2] ** 2)
    nx, ny, nz = r[0] / norm, r[1] / norm, r[2] / norm
    c = math.sqrt(max(0.0, (1.0 + nz) / 2.0))
    s = math.sqrt(max(0.0, (1.0 - nz) / 2.0))
    if s < 1e-15:
        return np.array([1.0, 0.0], dtype=complex)
    return np.array([c, s * np.exp(1j * math.atan2(ny, nx))], dtype=complex)


def round_qubit(amps: np.ndarray, q: int):
    """SDRP step of engine.py:464-488 on a copy: returns (phi, rest) or None
    when numerically degenerate."""
    amps = amps.copy()
    r = bloch_vector(amps, q)
    length = math.sqrt(r[0] ** 2 + r[1] ** 2 + r[2] ** 2)
    if length < 1e-12:
        u, phi = None, np.array([1.0, 0.0], dtype=complex)
    else:
        phi = bloch_to_state(r)
        u = np.array([[np.conj(phi[0]), np.conj(phi[1])], [-phi[1], phi[0]]], dtype=complex)
    if u is not None:
        apply_1q(amps, q, u)
    if probability(amps, q, 0) < 1e-12:
        return None
    project_and_renormalize(amps, q, 0)
    return phi, remove_qubit(amps, q)


def sample(amps: np.ndarray, rng, shots=None):
    """engine.py:613-615 / 648-650: rng.choice over |a|^2 normalised."""
    probs = np.abs(amps) ** 2
    probs /= probs.sum()
    return rng.choice(probs.size, size=shots, p=probs)


# ---------------------------------------------------------------------------
# dense circuit loop and DFT oracle (validate.py:41-111)
# ---------------------------------------------------------------------------

_X = np.array([[0, 1], [1, 0]], dtype=complex)


def dense_run(gates, amps: np.ndarray, gate_matrix, label_swap: bool = False, rng=None) -> np.ndarray:
    """validate.py:83-111 without the 2^26 cap (:86-87), in place on `amps`.

    label_swap=True skips SWAPs (engine.py:525-535 semantics); the caller then
    reads the result through the swapped labels (see `swap_permutation`)."""
    for g in gates:
        if g.name == "m":
            p1 = probability(amps, g.targets[0], 1)
            outcome = 1 if rng.random() < p1 else 0
            project_and_renormalize(amps, g.targets[0], outcome)
        elif g.name == "swap":
            if label_swap:
                continue
            a, b = g.targets
            apply_controlled(amps, (a,), (1,), b, _X)
            apply_controlled(amps, (b,), (1,), a, _X)
            apply_controlled(amps, (a,), (1,), b, _X)
        elif g.controls:
            apply_controlled(amps, g.controls, g.polarity, g.targets[0], gate_matrix(g.name, g.params))
        else:
            apply_1q(amps, g.targets[0], gate_matrix(g.name, g.params))
    return amps


def swap_permutation(gates, n: int) -> list[int]:
    """phys[label] after label-swapping every SWAP in `gates`."""
    phys = list(range(n))
    for g in gates:
        if g.name == "swap":
            a, b = g.targets
            phys[a], phys[b] = phys[b], phys[a]
    return phys


def dft_oracle(x) -> np.ndarray:
    """Radix-2 unitary DFT with positive exponent (validate.py:41-66)."""
    x = np.asarray(x, dtype=complex)
    n = x.size
    if n == 0 or n & (n - 1):
        raise ValueError(f"length must be a power of two, got {n}")
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    y = x[rev]
    half = 1
    while half < n:
        tw = np.exp(2j * np.pi * np.arange(half) / (2 * half))
        blocks = y.reshape(-1, 2 * half)
        even = blocks[:, :half].copy()
        odd = blocks[:, half:] * tw
        blocks[:, :half] = even + odd
        blocks[:, half:] = even - odd
        half *= 2
    return y / math.sqrt(n)


def qft_of_ghz(n: int, idx) -> np.ndarray:
    """Closed form of the QFT of (|0..0> + |1..1>)/sqrt(2):
    y_j = (1 + exp(2 pi i j (N-1)/N)) / sqrt(2N) = (1 + exp(-2 pi i j/N)) / sqrt(2N)."""
    N = float(1 << n)
    j = np.asarray(idx, dtype=np.float64)
    return (1.0 + np.exp(-2j * np.pi * j / N)) / math.sqrt(2.0 * N)


def dft_at(x: np.ndarray, idx) -> np.ndarray:
    """Direct DFT entries y_j = sum_k x_k e^{2 pi i jk/N}/sqrt(N) at a few j
    (an O(N) per index cross-check usable at any N)."""
    x = np.asarray(x, dtype=complex)
    N = x.size
    k = np.arange(N, dtype=np.int64)
    out = []
    for j in np.atleast_1d(idx):
        ph = np.exp(2j * np.pi * ((int(j) * k) % N).astype(np.float64) / N)
        out.append(np.dot(ph, x) / math.sqrt(N))
    return np.array(out)
