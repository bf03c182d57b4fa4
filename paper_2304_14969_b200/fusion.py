"""Gate-fusion planner for the fused dense executor.

Turns a circuit into a program for `k_sweep` (csrc/sk_fused.cu): a list of
sweeps, each one HBM read + write of the state, each holding stages of ops
applied on register-resident amplitudes.  The reference's counterpart is the
gate-by-gate loop `dense_reference` (validate.py:83-111), one NumPy pass per
gate; SWAPs become label permutations as in the engine (engine.py:525-535).

Lowering (per gate, on physical bits):
  * 1q / controlled gate with an exactly diagonal matrix (the reference's
    fast-path test, ket.py:136,153)          -> DIAG (needs no pairing)
  * otherwise                                -> MAT on its target
  * a run of consecutive diagonal ops is reordered freely (they commute);
    controlled phases sharing a target whose controls form a contiguous bit
    field with angles pi*s*2^(c-lo) collapse into ONE RAMP op
    exp(i*pi*s*F), F = (idx >> lo) & (2^k - 1): the QFT's fan-in of CPs.

Scheduling: op A may move ahead of op B iff neither acts non-diagonally on a
bit the other touches.  A sweep greedily takes every op (in order) that
commutes with all ops left behind and whose non-diagonal target fits the
tile (T bits, always including the lowest `low_bits` bits so warps stream
>= 256 contiguous bytes).  Inside a sweep, stages are packed the same way
with capacity NR register bits; the first and last stage keep their
register bits off the low bits so HBM loads and stores stay coalesced.
"""
from __future__ import annotations

import cmath
import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .circuit import Circuit, gate_matrix

MAT, DIAG, RAMP, QFT = _lib.SK_OP_MAT, _lib.SK_OP_DIAG, _lib.SK_OP_RAMP, _lib.SK_OP_QFT
MAX_STAGES = _lib.SK_MAX_STAGES

# kernel geometry per dtype (csrc/sk_fused.cu): register bits, max tile bits,
# low contiguous bits (256 B per warp access)
GEOMETRY = {"c64": dict(nreg=4, tile=11, low=4, qft_tile=12, qft_low=4, qft_nreg=4),
            "c128": dict(nreg=3, tile=10, low=4, qft_tile=11, qft_low=3, qft_nreg=4)}
# Measured on B200 (scripts/tune_qft.py): QFT-27 c64 1.10 ms at T=12/low=4
# (k_qft); c128 QFT windows use 4 register bits (16 amplitudes per thread):
# QFT-27 c128 2.44 ms in 3 sweeps at T=11/low=3 vs 2.98 ms in 4 sweeps with 3
# register bits at T=10/low=4; c64 5-bit QFT chunks (qft_nreg=5, 32
# amplitudes per thread, 2/2/3 stages at T=13) measured 1.18 ms vs 1.09 ms
# for 4-bit chunks at T=12 (half the occupancy costs more than the saved
# exchange); random 30x20 c64 384 ms at T=11/low=5 vs 467 ms at T=13/low=5 and
# c128 803 ms at T=10/low=4 vs 917 ms at T=12 (generic k_sweep: fewer, larger
# tiles lose occupancy to its ~110 registers per thread).  Round 2 (LEAN op
# tables in the parameter space, two tiles per CTA): random 30x20 c64
# 192.6 ms at T=11/low=4 (30 sweeps) vs 199.9 ms at low=5 (34 sweeps),
# 202.9 at T=10/low=4, 207.6 at T=12/low=4.


@dataclass
class Op:
    kind: int
    qubit: int
    m: tuple  # 8 doubles
    ctrl_mask: int = 0
    ctrl_val: int = 0
    nbits: int = 0
    src: int = -1  # index of the originating gate (diagnostics)
    pin: bool = False  # a phase of split_1q: keep its bit a register bit of its stage

    @property
    def tmask(self) -> int:
        """Bits acted on non-diagonally (and the bit of a pinned phase)."""
        if self.kind == QFT:
            return ((1 << self.nbits) - 1) << self.qubit
        return (1 << self.qubit) if self.kind == MAT or self.pin else 0

    @property
    def smask(self) -> int:
        """Every bit the op reads or acts on."""
        if self.kind == RAMP:
            s = ((1 << self.nbits) - 1) << self.qubit
        elif self.kind == QFT:  # reads the window above and everything below it
            s = (1 << (int(self.m[1]) + 1)) - 1
        else:
            s = 1 << self.qubit
        return s | self.ctrl_mask


def _m8(m) -> tuple:
    return (m[0, 0].real, m[0, 0].imag, m[0, 1].real, m[0, 1].imag,
            m[1, 0].real, m[1, 0].imag, m[1, 1].real, m[1, 1].imag)


def lower(circuit: Circuit, phys: list[int] | None = None):
    """Gates -> elementary ops on physical bits; returns (ops, phys) where
    phys[label] is the physical bit holding logical qubit `label` at the end."""
    n = circuit.width
    phys = list(range(n)) if phys is None else list(phys)
    ops: list[Op] = []
    for gi, g in enumerate(circuit.gates):
        if g.name == "m":
            raise ValueError("measurement gates are not fusable; split the circuit at them")
        if g.name == "swap":
            a, b = g.targets
            phys[a], phys[b] = phys[b], phys[a]
            continue
        m = gate_matrix(g.name, g.params)
        t = phys[g.targets[0]]
        cmask = cval = 0
        for c, pol in zip(g.controls, g.polarity):
            cmask |= 1 << phys[c]
            if pol:
                cval |= 1 << phys[c]
        diag = m[0, 1] == 0 and m[1, 0] == 0
        if diag and m[0, 0] == 1 and m[1, 1] == 1:
            continue  # identity (ket.py:154-158 skips both entries)
        ops.append(Op(DIAG if diag else MAT, t, _m8(m), cmask, cval, src=gi))
    return ops, phys


def merge_1q(ops: list[Op]) -> list[Op]:
    """Fold each uncontrolled 1q op into the previous uncontrolled 1q op on the
    same bit when no op in between touches that bit (they commute with
    everything else in between): m = m_later @ m_earlier.  In Sycamore-style
    layers a qubit outside every coupler of a layer carries two consecutive
    U3s (104 of 600 in random 30x20): one dense 2x2 pass instead of two."""
    out: list[Op] = []
    last: dict[int, int] = {}  # bit -> index in out of its open 1q op
    for op in ops:
        if op.ctrl_mask == 0 and op.kind in (MAT, DIAG):
            j = last.get(op.qubit)
            if j is not None:
                prev = out[j]
                a = np.array([[complex(op.m[0], op.m[1]), complex(op.m[2], op.m[3])],
                              [complex(op.m[4], op.m[5]), complex(op.m[6], op.m[7])]])
                b = np.array([[complex(prev.m[0], prev.m[1]), complex(prev.m[2], prev.m[3])],
                              [complex(prev.m[4], prev.m[5]), complex(prev.m[6], prev.m[7])]])
                m = a @ b
                diag = m[0, 1] == 0 and m[1, 0] == 0
                out[j] = Op(DIAG if diag else MAT, op.qubit, _m8(m), src=prev.src)
                continue
            last[op.qubit] = len(out)
            out.append(op)
            continue
        sm = op.smask
        for bit in list(last):
            if (sm >> bit) & 1:
                del last[bit]
        out.append(op)
    return out


SPLIT_1Q = bool(int(__import__("os").environ.get("SK_SPLIT_1Q", "1")))


def _zyz(m: np.ndarray):
    """m = e^{i g} diag(1, e^{i a}) [[c, -s], [s, c]] diag(1, e^{i b}) with
    c = |m00|, s = |m10| (m unitary); returns (g, a, b, c, s)."""
    c, s = abs(m[0, 0]), abs(m[1, 0])
    if c > 1e-300:
        g = cmath.phase(m[0, 0])
        b = cmath.phase(-m[0, 1]) - g if s > 1e-300 else cmath.phase(m[1, 1]) - g
        a = cmath.phase(m[1, 0]) - g if s > 1e-300 else 0.0
    else:  # anti-diagonal: pick g from m10 (a = 0)
        g = cmath.phase(m[1, 0])
        a = 0.0
        b = cmath.phase(-m[0, 1]) - g
    return g, a, b, c, s


def _splittable(op: Op) -> bool:
    """An uncontrolled dense 1q op that is neither real nor H-like (those keep
    their own fast paths)."""
    if op.kind != MAT or op.ctrl_mask:
        return False
    real = all(op.m[i] == 0.0 for i in (1, 3, 5, 7))
    bfly = op.m[0] == op.m[2] and op.m[1] == op.m[3] and op.m[4] == -op.m[6] and op.m[5] == -op.m[7]
    return not real and not bfly


def _mat(op: Op) -> np.ndarray:
    return np.array([[complex(op.m[0], op.m[1]), complex(op.m[2], op.m[3])],
                     [complex(op.m[4], op.m[5]), complex(op.m[6], op.m[7])]])


def split_1q(ops: list[Op]) -> list[Op]:
    """Carry the output phase of dense 1q gates to the next dense gate on the
    same bit.  U = e^{ig} diag(1, e^{ia}) R diag(1, e^{ib}) (R real): when
    every op between U and the next splittable gate V on that bit is
    diagonal on it (controlled phases, uses as a control, other bits),
    diag(1, e^{ia}) commutes up to V, so U is emitted as R diag(1, e^{ib}) —
    a 2x2 with a real first column, which k_sweep runs as a phase on a1 plus
    a real rotation (6 paired instructions per pair instead of 8) — and V
    absorbs the phase into its own input side.  The op count is unchanged;
    gates without such a successor stay full 2x2s (and carry the global
    phase).  Exact up to fp64 rounding (the fused-executor tests check it
    against the oracle)."""
    n = len(ops)
    # nxt[i]: for a splittable op i, True when the next op non-diagonal on its
    # bit is again a splittable op (its deferred phase has a consumer)
    nxt = [False] * n
    last: dict[int, int] = {}  # bit -> index of the next op non-diagonal on it (scanning backwards)
    for i in range(n - 1, -1, -1):
        op = ops[i]
        if _splittable(op):
            j = last.get(op.qubit)
            nxt[i] = j is not None and _splittable(ops[j])
        for q in _bits(op.tmask):
            last[q] = i
    out: list[Op] = []
    pend: dict[int, float] = {}
    gphase = 0.0
    full_idx = -1
    for i, op in enumerate(ops):
        if not _splittable(op):
            out.append(op)
            continue
        q = op.qubit
        m = _mat(op)
        if abs(abs(np.linalg.det(m)) - 1.0) > 1e-9 or np.max(np.abs(m.conj().T @ m - np.eye(2))) > 1e-9:
            m = m @ np.diag([1.0, cmath.exp(1j * pend.pop(q, 0.0))])  # not unitary: dense as given
            out.append(Op(MAT, q, _m8(m), src=op.src))
            continue
        g, a, b, c, s_ = _zyz(m)
        b += pend.pop(q, 0.0)
        eb = cmath.exp(1j * b)
        if nxt[i]:  # R diag(1, e^{ib}); diag(1, e^{ia}) moves on to the next gate on q
            pend[q] = a
            gphase += g
            out.append(Op(MAT, q, (c, 0.0, -s_ * eb.real, -s_ * eb.imag, s_, 0.0, c * eb.real, c * eb.imag),
                          src=op.src))
        else:  # the whole gate, with the phases it absorbed
            mm = cmath.exp(1j * g) * np.array([[c, -s_ * eb], [s_ * cmath.exp(1j * a), c * cmath.exp(1j * a) * eb]])
            out.append(Op(MAT, q, _m8(mm), src=op.src))
            full_idx = len(out) - 1
    assert not pend, "deferred phases must all be consumed"
    gw = _wrap(gphase)
    if gw != 0.0:
        if full_idx < 0:  # cannot happen (the last splittable gate on a bit is always full)
            raise AssertionError("no full gate to carry the global phase")
        o = out[full_idx]
        out[full_idx] = Op(MAT, o.qubit, _m8(cmath.exp(1j * gw) * _mat(o)), src=o.src)
    return out


def _wrap(a: float) -> float:
    return (a + math.pi) % (2 * math.pi) - math.pi


def _try_ramp(target: int, group: list[Op]) -> Op | None:
    """Collapse controlled phases diag(1, e^{i phi_c}) on `target` with single
    controls c (polarity 1) into one RAMP if the controls are a contiguous
    field and phi_c = pi * s * 2^(c - lo)."""
    if len(group) < 2:
        return None
    phis = {}
    for op in group:
        if op.ctrl_mask == 0 or op.ctrl_mask & (op.ctrl_mask - 1) or op.ctrl_val != op.ctrl_mask:
            return None
        if op.m[0] != 1.0 or op.m[1] != 0.0:
            return None
        c = op.ctrl_mask.bit_length() - 1
        if c in phis:
            return None
        phis[c] = math.atan2(op.m[7], op.m[6])
    lo, hi = min(phis), max(phis)
    if hi - lo + 1 != len(phis):
        return None
    s = phis[lo] / math.pi
    for c, phi in phis.items():
        if abs(_wrap(phi - math.pi * s * (1 << (c - lo)))) > 1e-12:
            return None
    return Op(RAMP, lo, (s, 0, 0, 0, 0, 0, 0, 0), 1 << target, 1 << target, nbits=hi - lo + 1,
              src=group[0].src)


def fuse_diagonal_runs(ops: list[Op]) -> list[Op]:
    """Within each maximal run of consecutive diagonal ops, collapse QFT-style
    controlled-phase fans into RAMP ops (diagonal ops commute, so the run may
    be regrouped by target)."""
    out: list[Op] = []
    i = 0
    while i < len(ops):
        if ops[i].kind != DIAG:
            out.append(ops[i])
            i += 1
            continue
        j = i
        while j < len(ops) and ops[j].kind == DIAG:
            j += 1
        run = ops[i:j]
        by_target: dict[int, list[Op]] = {}
        order: list[int] = []
        for op in run:
            if op.qubit not in by_target:
                by_target[op.qubit] = []
                order.append(op.qubit)
            by_target[op.qubit].append(op)
        for t in order:
            grp = by_target[t]
            ramp = _try_ramp(t, grp)
            out.extend([ramp] if ramp is not None else grp)
        i = j
    return out


def _pack(ops: list[Op], capacity: int, base_mask: int):
    """Greedy commutation-aware packing: take every op that commutes with all
    skipped ops and whose non-diagonal target fits `capacity` bits together
    with `base_mask`.  Returns (taken, skipped, mask)."""
    mask = base_mask
    taken, skipped = [], []
    sk_t = sk_s = 0
    for op in ops:
        t, s = op.tmask, op.smask
        if (t & sk_s) == 0 and (sk_t & s) == 0 and bin(mask | t).count("1") <= capacity:
            taken.append(op)
            mask |= t
        else:
            skipped.append(op)
            sk_t |= t
            sk_s |= s
    return taken, skipped, mask


@dataclass
class StagePlan:
    reg_bits: list[int]
    ops: list[Op] = field(default_factory=list)


@dataclass
class SweepPlan:
    tile_bits: list[int]
    stages: list[StagePlan]


@dataclass
class Plan:
    width: int
    dtype: str
    nreg: int
    sweeps: list[SweepPlan]
    phys: list[int]
    n_gates: int
    n_ops: int

    @property
    def order(self) -> list[int]:
        """`permute_qubits` order taking the physical result to label order."""
        return list(self.phys)


def _bits(mask: int) -> list[int]:
    out = []
    b = 0
    while mask:
        if mask & 1:
            out.append(b)
        mask >>= 1
        b += 1
    return out


def _stages_for(ops: list[Op], tile: list[int], nreg: int, low: int) -> list[StagePlan]:
    """Split a sweep's ops into register stages (commutation-aware greedy) and
    pad every stage to exactly nreg register bits."""
    stages: list[StagePlan] = []
    rest = list(ops)
    while rest:
        taken, rest, mask = _pack(rest, nreg, 0)
        stages.append(StagePlan(_bits(mask), taken))
    if not stages:
        stages.append(StagePlan([], []))
    low_mask = (1 << low) - 1
    tile_desc = sorted(tile, reverse=True)

    def pad(regs: list[int], avoid_low: bool) -> list[int]:
        regs = list(regs)
        for b in tile_desc:
            if len(regs) >= nreg:
                break
            if b not in regs and not (avoid_low and (1 << b) & low_mask):
                regs.append(b)
        for b in tile_desc:  # tiny tiles: fall back to any bit
            if len(regs) >= nreg:
                break
            if b not in regs:
                regs.append(b)
        return regs

    coalesce = len(tile) - nreg >= low  # enough thread bits to keep lanes on the low bits
    first_bad = coalesce and any((1 << b) & low_mask for b in stages[0].reg_bits)
    if first_bad:
        stages.insert(0, StagePlan([], []))
    last_bad = coalesce and any((1 << b) & low_mask for b in stages[-1].reg_bits)
    if last_bad:
        stages.append(StagePlan([], []))
    for i, st in enumerate(stages):
        edge = i == 0 or i == len(stages) - 1
        st.reg_bits = pad(st.reg_bits, avoid_low=edge and coalesce)
    return stages


def plan_ops(ops: list[Op], width: int, dtype: str = "c64", tile_bits: int | None = None,
             low_bits: int | None = None, phys=None, n_gates: int = 0) -> Plan:
    geo = GEOMETRY[dtype]
    nreg = geo["nreg"]
    T = min(tile_bits or geo["tile"], width)
    low = min(low_bits if low_bits is not None else geo["low"], T)
    if T < nreg:
        raise ValueError(f"width {width} too small for the fused kernel (needs >= {nreg})")
    base = (1 << low) - 1
    sweeps: list[SweepPlan] = []
    remaining = list(ops)
    while remaining:
        taken, skipped, mask = _pack(remaining, T, base)
        # fill the tile with the lowest unused bits (more coalescing, same cost)
        b = 0
        while bin(mask).count("1") < T:
            mask |= 1 << b
            b += 1
        tile = _bits(mask)
        stages = _stages_for(taken, tile, nreg, low)
        if len(stages) > MAX_STAGES:
            # keep the ops of the first stages only; the rest go back in order
            keep = []
            while True:
                st = _stages_for(taken[: len(keep) + 1], tile, nreg, low)
                if len(st) > MAX_STAGES:
                    break
                keep = taken[: len(keep) + 1]
            executed = {id(o) for o in keep}
            stages = _stages_for(keep, tile, nreg, low)
            remaining = [o for o in remaining if id(o) not in executed]
        else:
            remaining = skipped
        sweeps.append(SweepPlan(tile, stages))
    return Plan(width, dtype, nreg, sweeps, list(phys) if phys is not None else list(range(width)),
                n_gates, len(ops))


_H_M8 = _m8(gate_matrix("h"))


def match_qft(ops: list[Op], n: int) -> bool:
    """True when `ops` is exactly the n-qubit QFT body (build_qft without the
    final swaps): for j = n-1..0, H(j) then the fan of CP(pi/2^k) from j-k
    onto j (a RAMP over bits [0, j) with s = 2^-j; j = 1 is a single CP)."""
    i = 0
    for j in range(n - 1, -1, -1):
        if i >= len(ops):
            return False
        op = ops[i]
        if op.kind != MAT or op.qubit != j or op.ctrl_mask or max(abs(a - b) for a, b in zip(op.m, _H_M8)) > 0:
            return False
        i += 1
        if j >= 2:
            if i >= len(ops):
                return False
            r = ops[i]
            if (r.kind != RAMP or r.qubit != 0 or r.nbits != j or r.ctrl_mask != 1 << j or r.ctrl_val != 1 << j
                    or abs(r.m[0] - 2.0 ** -j) > 1e-13 * 2.0 ** -j):
                return False
            i += 1
        elif j == 1:
            if i >= len(ops):
                return False
            d = ops[i]
            want = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0, math.cos(math.pi / 2), math.sin(math.pi / 2))
            if (d.kind != DIAG or d.qubit != 1 or d.ctrl_mask != 1 or d.ctrl_val != 1
                    or max(abs(a - b) for a, b in zip(d.m, want)) > 1e-15):
                return False
            i += 1
    return i == len(ops)


def plan_qft(n: int, dtype: str = "c64", tile_bits: int | None = None, low_bits: int | None = None,
             phys=None, n_gates: int = 0, nreg: int | None = None) -> Plan:
    """Sweeps for the QFT body in FFT form: windows of target bits from the
    top (each at most T - low bits, the bottom window up to T bits), each
    window split into register chunks of NR bits; one QFT op per chunk."""
    geo = GEOMETRY[dtype]
    nreg = nreg or geo["qft_nreg"]
    if nreg > 4 and n < 2 * nreg:  # small registers: 4-bit chunks (the 5-bit kernel wants >= 2 chunks of room)
        nreg = 4
    T = min(tile_bits or geo["qft_tile"], n)
    low = min(low_bits if low_bits is not None else geo["qft_low"], T)
    windows = []
    hi = n - 1
    while hi >= 0:
        if hi + 1 <= T:  # bottom window: everything left fits one tile
            windows.append((0, hi))
            break
        k = T - low
        windows.append((hi - k + 1, hi))
        hi -= k
    sweeps = []
    for w_lo, w_hi in windows:
        tile_mask = ((1 << low) - 1) | (((1 << (w_hi - w_lo + 1)) - 1) << w_lo)
        b = 0
        while bin(tile_mask).count("1") < T:
            tile_mask |= 1 << b
            b += 1
        tile = _bits(tile_mask)
        stages = []
        K = w_hi - w_lo + 1
        sizes = [K % nreg or nreg] + [nreg] * ((K - (K % nreg or nreg)) // nreg)  # short chunk first
        c_hi = w_hi
        prev_hi = None
        for ci, size in enumerate(sizes):
            c_lo = c_hi - size + 1
            last = ci == len(sizes) - 1
            # pad bits must not be read by this chunk's phases: no earlier-chunk window
            # bits (entry twiddle) and no below-window bits when a twiddle reads L
            uses_l = (ci > 0) or (last and w_lo > 0)
            allowed = [x for x in sorted(tile, reverse=True)
                       if not (c_lo <= x <= w_hi) and not (uses_l and x < w_lo)]
            regs = list(range(c_lo, c_hi + 1))
            for pref in (lambda x: x >= low, lambda x: True):
                for x in allowed:
                    if len(regs) < nreg and x not in regs and pref(x):
                        regs.append(x)
            if len(regs) < nreg:
                raise ValueError("QFT window chunk cannot be padded")
            op = Op(QFT, c_lo, (float(w_lo), float(w_hi), float(prev_hi if prev_hi is not None else -1),
                                0, 0, 0, 0, 0), nbits=size)
            stages.append(StagePlan(sorted(regs), [op]))
            prev_hi = c_hi
            c_hi = c_lo - 1
        low_mask = (1 << low) - 1
        if len(tile) - nreg >= low and any((1 << x) & low_mask for x in stages[-1].reg_bits):
            stages.append(StagePlan(sorted(tile, reverse=True)[:nreg], []))  # store stage: lanes on low bits
        if len(stages) > MAX_STAGES:
            raise ValueError("QFT window needs too many stages")
        sweeps.append(SweepPlan(tile, stages))
    return Plan(n, dtype, nreg, sweeps, list(phys) if phys is not None else list(range(n)), n_gates,
                sum(len(st.ops) for sp in sweeps for st in sp.stages))


def plan_circuit(circuit: Circuit, dtype: str = "c64", tile_bits: int | None = None,
                 low_bits: int | None = None, fuse: bool = True, qft: bool = True, qft_nreg: int | None = None) -> Plan:
    ops, phys = lower(circuit)
    if fuse:
        ops = fuse_diagonal_runs(ops)
    geo = GEOMETRY[dtype]
    if qft and fuse and circuit.width >= geo["nreg"] + 1 and match_qft(ops, circuit.width):
        try:
            return plan_qft(circuit.width, dtype, tile_bits, low_bits, phys, len(circuit.gates), qft_nreg)
        except ValueError:
            pass  # geometry the QFT form cannot pad: fall back to generic sweeps
    if fuse:
        ops = merge_1q(ops)
        if SPLIT_1Q:
            ops = split_1q(ops)
    return plan_ops(ops, circuit.width, dtype, tile_bits, low_bits, phys, len(circuit.gates))


def to_c(plan: Plan):
    """Plan -> (SkSweep array, SkOp array) for sk_program_create."""
    flat: list[Op] = []
    sweeps = (_lib.SkSweep * len(plan.sweeps))()
    for si, sp in enumerate(plan.sweeps):
        cs = sweeps[si]
        cs.ntile = len(sp.tile_bits)
        cs.nreg = plan.nreg
        for i, b in enumerate(sp.tile_bits):
            cs.tile_bits[i] = b
        cs.nstages = len(sp.stages)
        for s, st in enumerate(sp.stages):
            for p, b in enumerate(st.reg_bits):
                cs.reg_bits[s][p] = b
            cs.op_begin[s] = len(flat)
            flat.extend(st.ops)
        cs.op_begin[len(sp.stages)] = len(flat)
    ops = (_lib.SkOp * max(1, len(flat)))()
    for i, op in enumerate(flat):
        co = ops[i]
        co.kind = op.kind
        co.qubit = op.qubit
        co.nbits = op.nbits
        co.ctrl_mask = op.ctrl_mask
        co.ctrl_val = op.ctrl_val
        for k in range(8):
            co.m[k] = float(op.m[k])
    return sweeps, ops, len(flat)


# ---------------------------------------------------------------------------
# host-side interpreter of a plan's op semantics (used by the CPU tests to
# check lowering, RAMP fusion and commutation-based reordering; the device
# kernel is checked against the oracle on the GPU)
# ---------------------------------------------------------------------------
def apply_op_numpy(amps: np.ndarray, op: Op) -> None:
    n = amps.size
    idx = np.arange(n, dtype=np.int64)
    if op.kind == QFT:  # one register chunk of a QFT window, FFT form (see csrc/sk_fused.cu)
        w_lo, w_hi, prev_hi = int(op.m[0]), int(op.m[1]), int(op.m[2])
        c_lo, c_hi = op.qubit, op.qubit + op.nbits - 1
        bit = lambda q: (idx >> q) & 1  # noqa: E731
        L = idx & ((1 << w_lo) - 1)
        if c_hi < w_hi:  # entry: cross phases with earlier chunks + their deferred below-window phase
            th_all = sum(bit(j) * 2.0 ** -j for j in range(c_hi + 1, w_hi + 1))
            th_new = sum(bit(j) * 2.0 ** -j for j in range(c_hi + 1, prev_hi + 1))
            cur = sum(bit(i) << i for i in range(c_lo, c_hi + 1))
            amps *= np.exp(1j * np.pi * np.mod(th_all * cur + th_new * L, 2.0))
        h = 1 / math.sqrt(2)
        for j in range(c_hi, c_lo - 1, -1):
            i0 = idx[bit(j) == 0]
            i1 = i0 | (1 << j)
            a0, a1 = amps[i0].copy(), amps[i1].copy()
            amps[i0] = h * (a0 + a1)
            amps[i1] = h * (a0 - a1)
            inner = sum(bit(i) * 2.0 ** (i - j) for i in range(c_lo, j))
            amps *= np.where(bit(j) == 1, np.exp(1j * np.pi * inner), 1.0)
        if c_lo == w_lo and w_lo > 0:  # window end: this chunk's deferred below-window phase
            amps *= np.exp(1j * np.pi * np.mod(L * sum(bit(i) * 2.0 ** -i for i in range(c_lo, c_hi + 1)), 2.0))
        return
    sel = (idx & op.ctrl_mask) == op.ctrl_val
    if op.kind == MAT:
        bit = 1 << op.qubit
        i0 = idx[sel & ((idx & bit) == 0)]
        i1 = i0 | bit
        m = op.m
        m00, m01, m10, m11 = complex(m[0], m[1]), complex(m[2], m[3]), complex(m[4], m[5]), complex(m[6], m[7])
        a0, a1 = amps[i0].copy(), amps[i1].copy()
        amps[i0] = m00 * a0 + m01 * a1
        amps[i1] = m10 * a0 + m11 * a1
    elif op.kind == DIAG:
        m = op.m
        d = np.where((idx >> op.qubit) & 1, complex(m[6], m[7]), complex(m[0], m[1]))
        amps[sel] *= d[sel]
    else:
        f = (idx >> op.qubit) & ((1 << op.nbits) - 1)
        x = np.mod(op.m[0] * f.astype(np.float64), 2.0)
        amps[sel] *= np.exp(1j * np.pi * x[sel])


def run_plan_numpy(plan: Plan, amps: np.ndarray) -> np.ndarray:
    for sp in plan.sweeps:
        for st in sp.stages:
            for op in st.ops:
                if op.kind == MAT:
                    assert op.qubit in st.reg_bits and op.qubit in sp.tile_bits
                if op.kind == QFT:
                    assert set(range(op.qubit, op.qubit + op.nbits)) <= set(st.reg_bits)
                apply_op_numpy(amps, op)
    return amps
