"""Gate-fusion planner (host logic, CPU only): the planned op order applied
with NumPy equals the oracle's gate-by-gate dense loop; plans respect the
kernel's structural contract; QFT collapses to ceil-few sweeps."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import ket_oracle as O
from paper_2304_14969_b200 import fusion
from paper_2304_14969_b200.circuit import (Circuit, build_ghz, build_qft, build_random_circuit, cp, cx, gate_matrix,
                                           h, rz, swap, u3)

from conftest import random_state


def check_structure(plan: fusion.Plan):
    geo = fusion.GEOMETRY[plan.dtype]
    for sp in plan.sweeps:
        assert sp.tile_bits == sorted(set(sp.tile_bits))
        assert len(sp.tile_bits) <= max(geo["tile"], geo["qft_tile"], 13 if plan.dtype == "c64" else 12)
        assert 1 <= len(sp.stages) <= fusion.MAX_STAGES
        for st in sp.stages:
            assert len(st.reg_bits) == plan.nreg == len(set(st.reg_bits))
            assert set(st.reg_bits) <= set(sp.tile_bits)
            for op in st.ops:
                if op.kind == fusion.MAT:
                    assert op.qubit in st.reg_bits


def run_planned(c, x, dtype="c64", **kw):
    plan = fusion.plan_circuit(c, dtype=dtype, **kw)
    check_structure(plan)
    out = fusion.run_plan_numpy(plan, x.copy())
    return O.permute_qubits(out, plan.order), plan


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_qft_plan_equals_oracle(rng, dtype):
    for n in range(4, 13):
        x = random_state(n, rng)
        got, plan = run_planned(build_qft(n), x, dtype, tile_bits=min(n, 7), low_bits=2)
        want = O.dense_run(build_qft(n).gates, x.copy(), gate_matrix)
        assert np.max(np.abs(got - want)) < 1e-12, n


def test_qft_ramp_fusion_collapses_fans():
    ops, _ = fusion.lower(build_qft(10))
    fused = fusion.fuse_diagonal_runs(ops)
    ramps = [o for o in fused if o.kind == fusion.RAMP]
    assert len(ramps) == 8  # targets j = 9..2 (j = 1 has a single CP)
    assert sum(o.kind == fusion.MAT for o in fused) == 10


def test_qft27_is_three_sweeps():
    plan = fusion.plan_circuit(build_qft(27), dtype="c64")
    check_structure(plan)
    assert len(plan.sweeps) == 3
    plan64 = fusion.plan_circuit(build_qft(27), dtype="c128")
    check_structure(plan64)
    assert len(plan64.sweeps) == 3  # fp64 QFT windows: 4 register bits, 11-bit tiles (scripts/tune_qft.py)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_circuit_plan_equals_oracle(seed):
    c = build_random_circuit(10, 8, seed)
    x = np.zeros(1 << 10, complex)
    x[0] = 1
    got, plan = run_planned(c, x, "c64", tile_bits=8, low_bits=3)
    want = O.dense_run(c.gates, x.copy(), gate_matrix)
    assert np.max(np.abs(got - want)) < 1e-12
    assert len(plan.sweeps) < len(c.gates)


def test_mixed_gates_with_swaps_and_controls(rng):
    n = 9
    gates = [h(0), cx(0, 5), swap(1, 7), u3(0.3, 0.2, 0.1, 7), rz(0.4, 3), cp(0.7, 3, 8), swap(0, 8),
             cx(8, 2), h(4), cp(math.pi / 2, 4, 6), cp(math.pi / 4, 3, 6), cp(math.pi / 8, 2, 6)]
    from paper_2304_14969_b200.circuit import Gate
    gates.append(Gate("x", (1,), controls=(2, 6), polarity=(1, 0)))
    c = Circuit(n, tuple(gates))
    x = random_state(n, rng)
    got, plan = run_planned(c, x, "c128", tile_bits=6, low_bits=2)
    want = O.dense_run(c.gates, x.copy(), gate_matrix)
    assert np.max(np.abs(got - want)) < 1e-12


def test_ghz_and_tiny_tiles(rng):
    for n in (4, 5, 6):
        c = build_ghz(n)
        x = np.zeros(1 << n, complex)
        x[0] = 1
        got, _ = run_planned(c, x, "c64", tile_bits=4, low_bits=0)
        want = O.dense_run(c.gates, x.copy(), gate_matrix)
        assert np.max(np.abs(got - want)) < 1e-14


def test_to_c_roundtrip():
    plan = fusion.plan_circuit(build_qft(16), dtype="c64")
    sweeps, ops, nops = fusion.to_c(plan)
    assert nops == sum(len(st.ops) for sp in plan.sweeps for st in sp.stages)
    assert sweeps[0].ntile == fusion.GEOMETRY["c64"]["qft_tile"] and sweeps[-1].op_begin[sweeps[-1].nstages] == nops
    assert all(sweeps[i].nreg == plan.nreg for i in range(len(plan.sweeps)))


def test_qft_five_register_bit_chunks():
    """c64 QFT windows can use 5 register bits (32 amplitudes per thread):
    windows of 9 bits split [4, 5], QFT-27 = 3 sweeps of 2/2/3 stages."""
    plan = fusion.plan_circuit(build_qft(27), dtype="c64", tile_bits=13, low_bits=4, qft_nreg=5)
    assert plan.nreg == 5 and [len(sp.stages) for sp in plan.sweeps] == [2, 2, 3]
    assert [op.nbits for st in plan.sweeps[0].stages for op in st.ops] == [4, 5]


@pytest.mark.parametrize("seed", [3, 4])
def test_split_1q_keeps_op_count_and_exactness(rng, seed):
    """split_1q (phase carried to the next dense gate on the bit): same op
    count, most dense gates in real-first-column form, and the ops applied in
    order equal the unsplit ops to fp64 rounding on a random state."""
    c = build_random_circuit(9, 10, seed)
    ops, _ = fusion.lower(c)
    ops = fusion.merge_1q(fusion.fuse_diagonal_runs(ops))
    split = fusion.split_1q(ops)
    assert len(split) == len(ops)
    dense = [o for o in split if o.kind == fusion.MAT and not o.ctrl_mask]
    realcol = [o for o in dense if o.m[1] == 0.0 and o.m[5] == 0.0 and o.m[0] >= 0 and o.m[4] >= 0]
    assert len(realcol) >= len(dense) // 2
    x = random_state(9, rng)
    a, b = x.copy(), x.copy()
    for o in ops:
        fusion.apply_op_numpy(a, o)
    for o in split:
        fusion.apply_op_numpy(b, o)
    assert np.max(np.abs(a - b)) < 1e-12
