"""Fused dense executor: the GPU analogue of `dense_reference`.

`dense_reference(c, initial, rng)` (validate.py:83-111) runs a circuit gate
by gate with one NumPy pass per gate.  Here a circuit is planned once
(fusion.py) into a handful of sweeps of the fused kernel and replayed on a
device-resident state; SWAPs are label permutations (engine.py:525-535) and
the result is permuted back to label order only when read out.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib, fusion
from .circuit import Circuit
from .errors import MemoryBudgetError
from .ket import DenseKet, get_default_device, get_default_dtype, permute_qubits


class Program:
    """A planned circuit uploaded to the device (sk_program)."""

    def __init__(self, plan: fusion.Plan, device: int | None = None):
        self.plan = plan
        self.device = get_default_device() if device is None else device
        sweeps, ops, nops = fusion.to_c(plan)
        self._keep = (sweeps, ops)
        h = C.c_void_p()
        _lib.call("sk_program_create", plan.width, _lib.DTYPES[plan.dtype], self.device, sweeps, len(plan.sweeps),
                  ops, nops, C.byref(h))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.sk_program_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def n_sweeps(self) -> int:
        return len(self.plan.sweeps)

    def bytes_per_sweep(self) -> int:
        """Algorithmic HBM bytes of one sweep: read + write of 2^n amplitudes."""
        elem = 8 if self.plan.dtype == "c64" else 16
        return 2 * (1 << self.plan.width) * elem

    def run(self, state: DenseKet, first: int = 0, count: int = -1) -> None:
        if state.width != self.plan.width or state.dtype != self.plan.dtype:
            raise ValueError(f"program planned for width {self.plan.width} {self.plan.dtype}, "
                             f"state is width {state.width} {state.dtype}")
        _lib.call("sk_program_run", state._h, self._h, first, count)

    def set_phase_index(self, shift: int, value: int) -> None:
        """Run as the top layers of a larger QFT whose low `shift` qubits are
        the constant `value` (one-exchange sharded QFT; QFT-window programs)."""
        _lib.call("sk_program_set_phase_index", self._h, shift, value)

    def run_handle(self, handle, first: int = 0, count: int = -1) -> None:
        """Run on a raw sk_state handle (e.g. an sk_wrap view over a torch /
        NCCL buffer); the C side checks width, dtype and device."""
        _lib.call("sk_program_run", handle, self._h, first, count)


def compile_circuit(circuit: Circuit, dtype: str | None = None, device: int | None = None, **plan_kw) -> Program:
    dtype = dtype or get_default_dtype()
    return Program(fusion.plan_circuit(circuit, dtype=dtype, **plan_kw), device)


def _run_segment(gates, width, state: DenseKet, phys: list[int], dtype: str, device) -> list[int]:
    if not gates:
        return phys
    nreg = fusion.GEOMETRY[dtype]["nreg"]
    if width < nreg:  # tiny registers: per-gate kernels (still on the device)
        from .circuit import gate_matrix
        for g in gates:
            if g.name == "swap":
                a, b = g.targets
                phys[a], phys[b] = phys[b], phys[a]
            elif g.controls:
                state.apply_controlled(tuple(phys[c] for c in g.controls), g.polarity, phys[g.targets[0]],
                                       gate_matrix(g.name, g.params))
            else:
                state.apply_1q(phys[g.targets[0]], gate_matrix(g.name, g.params))
        return phys
    ops, phys = fusion.lower(Circuit(width, tuple(gates)), phys)
    ops = fusion.fuse_diagonal_runs(ops)
    if not ops:
        return phys
    plan = None
    if fusion.match_qft(ops, width):  # the QFT body: FFT-form windows
        try:
            plan = fusion.plan_qft(width, dtype, phys=phys)
        except ValueError:
            plan = None
    if plan is None:
        plan = fusion.plan_ops(fusion.merge_1q(ops), width, dtype, phys=phys)
    Program(plan, device).run(state)
    return phys


def dense_reference(c: Circuit, initial: DenseKet | None = None, rng=None, *, dtype: str | None = None,
                    device: int | None = None, budget: int | None = None) -> DenseKet:
    """Plain dense simulation of `c` on the device (validate.py:83-111).

    Same arguments and errors as the reference (ValueError on width mismatch
    or an 'm' gate without rng); the amplitude budget defaults to what fits
    in device memory instead of the reference's CPU cap of 2^26.
    Measurements draw `rng.random()` exactly like the reference (:95-100)."""
    dtype = dtype or (initial.dtype if initial is not None else get_default_dtype())
    if budget is not None and (1 << c.width) > budget:
        raise MemoryBudgetError(1 << c.width, budget)
    if initial is None:
        state = DenseKet(c.width, dtype=dtype, device=device)
    else:
        if initial.width != c.width:
            raise ValueError("initial state width mismatch")
        state = initial.copy() if initial.dtype == dtype else DenseKet(c.width, initial.amps, dtype=dtype)
    if any(g.name == "m" for g in c.gates) and rng is None:
        raise ValueError("circuit contains measurements; pass an rng")
    phys = list(range(c.width))
    seg: list = []
    for g in c.gates:
        if g.name != "m":
            seg.append(g)
            continue
        phys = _run_segment(seg, c.width, state, phys, dtype, device)
        seg = []
        q = phys[g.targets[0]]
        p1 = state.probability(q, 1)
        outcome = 1 if rng.random() < p1 else 0
        state.project_and_renormalize(q, outcome)
    phys = _run_segment(seg, c.width, state, phys, dtype, device)
    if phys != list(range(c.width)):
        state = permute_qubits(state, phys)
    return state
