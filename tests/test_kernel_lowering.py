"""Host-side lowering of fused programs into kernel ops (sk_program_lower,
no device needed), emulated with NumPy exactly as k_sweep applies them
(element masks, thread predicates, butterflies, folded fixed-point phases),
must reproduce the oracle's gate-by-gate dense loop.  CPU only."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import pytest

from oracle import ket_oracle as O
from paper_2304_14969_b200 import _lib, fusion
from paper_2304_14969_b200.circuit import (Circuit, Gate, build_qft, build_random_circuit, cp, cx, gate_matrix, h,
                                           rz, swap, u3)

from conftest import random_state

K_MAT, K_MATR, K_PHASE, K_TPHASE, K_BFLY, K_QFTS = range(6)
F_TPRED, F_QMASK, F_C0REAL, F_FOLD, F_TABLE, F_C0ONE = 1, 2, 4, 8, 16, 32
F_ENTRY, F_END, F_SCALE = 64, 128, 256
NS = _lib.SK_MAX_STAGES + 1


def lower(plan: fusion.Plan):
    sweeps, ops, nops = fusion.to_c(plan)
    cap = 64 * max(1, nops) + 64
    ints = (C.c_int64 * (12 * cap))()
    reals = (C.c_double * (24 * cap))()
    count = C.c_int()
    stage_ops = (C.c_int * (NS * len(plan.sweeps)))()
    _lib.call("sk_program_lower", plan.width, _lib.DTYPES[plan.dtype], sweeps, len(plan.sweeps), ops, nops, ints,
              reals, cap, C.byref(count), stage_ops)
    n = count.value
    I = np.frombuffer(ints, dtype=np.int64)[: 12 * n].reshape(n, 12)
    Rl = np.frombuffer(reals, dtype=np.float64)[: 24 * n].reshape(n, 24)
    return I, Rl, np.frombuffer(stage_ops, dtype=np.int32).reshape(len(plan.sweeps), NS)


def tau(turn, gthr, lo, fmask):
    f = (gthr >> np.uint64(lo)) & np.uint64(fmask)
    t = f * np.uint64(turn & 0xFFFFFFFFFFFFFFFF)  # wraps mod 2^64 like the kernel
    return np.exp(2j * np.pi * (t.astype(np.float64) / 2.0 ** 64))


def brev64(x):
    out = np.zeros_like(x)
    for b in range(64):
        out |= ((x >> np.uint64(b)) & np.uint64(1)) << np.uint64(63 - b)
    return out


def turn_phase(t):
    return np.exp(2j * np.pi * (t.astype(np.float64) / 2.0 ** 64))


def qft_chunk(amps, g, gthr, regs, e_of, slot, lo, nbits, flags, tmask, tval, qmask, scale):
    """K_QFTS exactly as the kernel computes it (wrapping uint64 turns)."""
    u64 = lambda v: np.uint64(v & (2**64 - 1))  # noqa: E731
    top, L = slot, nbits
    layer_slots = range(top - L + 1, top + 1)
    lv = gthr & u64(qmask)
    scaled = not (flags & F_SCALE)
    if flags & F_ENTRY:
        th_all, th_new = brev64(gthr & u64(tmask)), brev64(gthr & u64(tval))
        t = th_new * lv
        for p in layer_slots:
            t = t + np.where((e_of >> p) & 1, th_all << u64(lo + p - (top - L + 1)), np.uint64(0)).astype(np.uint64)
        here = not scaled and not (flags & F_END)
        amps *= turn_phase(t) * (scale if here else 1.0)
        scaled = scaled or here
    for P in range(top, top - L, -1):
        q = regs[P]
        i0 = np.nonzero(((g >> np.uint64(q)) & np.uint64(1)) == 0)[0]
        i1 = i0 | (1 << q)
        a0, a1 = amps[i0].copy(), amps[i1].copy()
        k16 = np.zeros(i0.size, dtype=np.int64)
        for p in range(top - L + 1, P):
            k16 += ((e_of[i0] >> p) & 1) << (4 - (P - p))
        amps[i0] = a0 + a1
        amps[i1] = (a0 - a1) * np.exp(1j * np.pi * k16 / 16)
    if flags & F_END:
        t = np.zeros_like(gthr)
        for p in layer_slots:
            t = t + np.where((e_of >> p) & 1, lv << u64(63 - (lo + p - (top - L + 1))), np.uint64(0)).astype(np.uint64)
        amps *= turn_phase(t) * (1.0 if scaled else scale)
        scaled = True
    if not scaled:
        amps *= scale


def emulate(plan: fusion.Plan, amps: np.ndarray, pshift: int = 0, pconst: int = 0) -> np.ndarray:
    """Run the lowered kernel ops in NumPy.  pshift/pconst mirror
    sk_program_set_phase_index (phase_shifted in csrc/sk_fused.cu): QFT chunk
    phases see the index (i << pshift) | pconst."""
    I, Rl, stage_ops = lower(plan)
    n = plan.width
    g = np.arange(1 << n, dtype=np.uint64)
    for si, sp in enumerate(plan.sweeps):
        for st, st_plan in enumerate(sp.stages):
            regs = st_plan.reg_bits
            regmask = sum(1 << q for q in regs)
            e_of = np.zeros(1 << n, dtype=np.int64)
            for p, q in enumerate(regs):
                e_of |= (((g >> np.uint64(q)) & np.uint64(1)).astype(np.int64)) << p
            gthr = g & np.uint64(~regmask & ((1 << 64) - 1))
            for k in range(stage_ops[si, st], stage_ops[si, st + 1]):
                kind, slot, pat, emask, flags, lo, nbits, tmask, tval, qmask, turn, fmask = (int(v) for v in I[k])
                m = Rl[k]
                if kind == K_QFTS:
                    if pshift:
                        tmask, tval, lo = tmask << pshift, tval << pshift, lo + pshift
                        qmask = (qmask << pshift) | ((1 << pshift) - 1)
                        if flags & F_SCALE:
                            flags |= F_END
                    gph = (gthr << np.uint64(pshift)) | np.uint64(pconst)
                    qft_chunk(amps, g, gph, regs, e_of, slot, lo, nbits, flags, tmask, tval, qmask, m[0])
                    continue
                ok = np.ones(1 << n, dtype=bool)
                if flags & F_TPRED:
                    ok = (gthr & np.uint64(tmask & (2**64 - 1))) == np.uint64(tval & (2**64 - 1))
                inmask = ((emask >> e_of) & 1).astype(bool) & ok
                if kind in (K_PHASE, K_TPHASE):
                    if kind == K_PHASE:
                        c = np.full(1 << n, complex(m[0], m[1]))
                        if flags & F_QMASK:
                            c = np.where((gthr & np.uint64(qmask)) != 0, complex(m[2], m[3]), c)
                    else:
                        c = tau(turn, gthr, lo, fmask)
                    amps[inmask] *= c[inmask]
                else:
                    q = regs[slot]
                    base = inmask & (((g >> np.uint64(q)) & np.uint64(1)) == 0)
                    i0 = np.nonzero(base)[0]
                    i1 = i0 | (1 << q)
                    a0, a1 = amps[i0].copy(), amps[i1].copy()
                    if kind == K_BFLY:
                        c0 = complex(m[0], m[1])
                        c1 = np.full(i0.size, complex(m[4], m[5]))
                        if flags & F_FOLD:
                            c1 = c1 * tau(turn, gthr[i0], lo, fmask)
                        if flags & F_TABLE:
                            e0 = e_of[i0]
                            kk = (e0 & ((1 << slot) - 1)) | ((e0 >> (slot + 1)) << slot)
                            tw = m[8::2] + 1j * m[9::2]
                            c1 = c1 * tw[kk]
                        amps[i0] = (a0 + a1) if flags & F_C0ONE else c0 * (a0 + a1)
                        amps[i1] = c1 * (a0 - a1)
                    else:
                        m00, m01 = complex(m[0], m[1]), complex(m[2], m[3])
                        m10, m11 = complex(m[4], m[5]), complex(m[6], m[7])
                        if flags & F_FOLD:
                            t = tau(turn, gthr[i0], lo, fmask)
                            m10, m11 = m10 * t, m11 * t
                        amps[i0] = m00 * a0 + m01 * a1
                        amps[i1] = m10 * a0 + m11 * a1
    return O.permute_qubits(amps, plan.order)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [5, 9, 14])
def test_qft_lowering(rng, dtype, n):
    x = random_state(n, rng)
    plan = fusion.plan_circuit(build_qft(n), dtype=dtype, tile_bits=min(n, 8), low_bits=min(3, n - 4), qft=False)
    got = emulate(plan, x.copy())
    assert np.max(np.abs(got - O.dft_oracle(x))) < 1e-12


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,tile,low", [(9, 7, 2), (12, 8, 3), (14, 10, 4), (15, 13, 5)])
def test_qft_fft_form_lowering(rng, dtype, n, tile, low):
    """The QFT-window (FFT-form) kernel path: chunk ops, fixed-point entry and
    end twiddles, compile-time internal twiddles, deferred scale."""
    x = random_state(n, rng)
    t = min(tile, fusion.GEOMETRY[dtype]["tile"])
    plan = fusion.plan_circuit(build_qft(n), dtype=dtype, tile_bits=t, low_bits=low)
    assert all(op.kind == fusion.QFT for sp in plan.sweeps for st in sp.stages for op in st.ops)
    I, _, _ = lower(plan)
    assert set(int(v) for v in I[:, 0]) == {K_QFTS}
    got = emulate(plan, x.copy())
    assert np.max(np.abs(got - O.dft_oracle(x))) < 1e-12


@pytest.mark.parametrize("n,G", [(9, 1), (11, 2), (13, 3)])
def test_phase_shifted_qft_windows(rng, n, G):
    """A QFT-window program for the top n-G qubits, run with phase index
    (i << G) | r on the slab whose low G qubits equal r, equals layers
    n-1..G of the n-qubit QFT (H(j) plus every CP onto j) restricted to that
    slab: the rank-constant CPs fold into the windows' twiddles."""
    x = random_state(n, rng)
    want = x.copy()
    for gt in build_qft(n).gates:
        if gt.name == "swap":
            continue
        j = gt.targets[0]
        if j < G:
            break  # layers G-1 .. 0 are the tail, run after the exchange
        O.dense_run((gt,), want, gate_matrix)
    plan = fusion.plan_qft(n - G, "c128", tile_bits=min(n - G, 8), low_bits=3)
    for r in range(1 << G):
        slab = x[r::1 << G].copy()
        got = emulate(plan, slab, pshift=G, pconst=r)
        assert np.max(np.abs(got - want[r::1 << G])) < 1e-12


def test_qft_lowering_uses_butterflies_and_folds():
    plan = fusion.plan_circuit(build_qft(16), dtype="c64", qft=False)
    I, _, _ = lower(plan)
    kinds = list(I[:, 0])
    assert kinds.count(K_BFLY) == 16
    assert kinds.count(K_TPHASE) == 0  # every RAMP's thread part folded into its H
    assert sum(1 for r in I if r[0] == K_PHASE and r[2] < 0) == 0  # all phases hit a specialised pattern
    # register-part phases ride in the butterflies' twiddle tables: only the
    # per-sweep deferred 1/sqrt(2)^L scalars (pattern 0) and the lone CP(0,1)
    # (a one-gate fan, not a RAMP) remain as phase ops
    assert sum(1 for r in I if r[0] == K_PHASE and r[2] == 0) == len(plan.sweeps)
    assert kinds.count(K_PHASE) == len(plan.sweeps) + 1


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_random_circuit_lowering(dtype):
    c = build_random_circuit(11, 6, 9)
    x = np.zeros(1 << 11, complex)
    x[0] = 1
    plan = fusion.plan_circuit(c, dtype=dtype, tile_bits=8, low_bits=3)
    got = emulate(plan, x)
    want = O.dense_run(c.gates, np.eye(1, 1 << 11, dtype=complex).ravel(), gate_matrix)
    assert np.max(np.abs(got - want)) < 1e-12


def test_mixed_controls_phases_and_general_ramps(rng):
    n = 10
    gates = [h(0), cx(0, 9), swap(1, 8), u3(0.3, 0.2, 0.1, 8), rz(0.4, 3), cp(0.7, 3, 9),
             Gate("y", (5,), controls=(2, 7), polarity=(1, 0)), Gate("z", (6,), controls=(1, 4), polarity=(0, 1)),
             h(4), Gate("p", (2,), (0.9,), controls=(8,), polarity=(0,))]
    gates += [cp(-0.37 * (1 << k), 6 - k, 6) for k in range(1, 6)]  # a general (non-dyadic) ramp
    gates += [cp(math.pi / (1 << k), 9 - k, 9) for k in range(1, 4)] + [h(9), h(6)]
    c = Circuit(n, tuple(gates))
    x = random_state(n, rng)
    want = O.dense_run(c.gates, x.copy(), gate_matrix)
    for dtype in ("c64", "c128"):
        plan = fusion.plan_circuit(c, dtype=dtype, tile_bits=7, low_bits=2)
        got = emulate(plan, x.copy())
        assert np.max(np.abs(got - want)) < 1e-12
