"""Every fast-path opcode of the generic fused sweep (`k_sweep<..., LEAN>`,
csrc/sk_fused.cu `lean_op`) against the oracle's gate-by-gate dense loop:
dense 2x2 (MAT, MATT, MATQ), X couplers as register swaps (SWAPT / SWAPQ),
Y couplers as swaps with +-i (YSWAPT / YSWAPQ), CZ-type couplers as sign
flips (SIGN) and general controlled phases (PHASE) — each with its control
on a register slot, a thread bit and a bit outside the tile, over several
tile geometries.  Tolerances are north_star's (1e-12 c128, 1e-5 c64)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import ket_oracle as O
from paper_2304_14969_b200 import fusion
from paper_2304_14969_b200.circuit import Circuit, ax, ay, az, cp, cx, cy, cz, gate_matrix, u3
from paper_2304_14969_b200.executor import compile_circuit
from paper_2304_14969_b200.ket import DenseKet, permute_qubits

from conftest import random_state

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 1e-5}
COUPLERS = (cx, cy, cz, ax, ay, az)


def coupler_circuit(n: int, n_gates: int, seed: int, phase_frac: float = 0.1) -> Circuit:
    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(n_gates):
        r = rng.random()
        a, b = (int(v) for v in rng.choice(n, 2, replace=False))
        if r < 0.35:
            gates.append(u3(*rng.uniform(0, 2 * math.pi, 3), a))
        elif r < 0.35 + phase_frac:
            gates.append(cp(float(rng.uniform(0, 2 * math.pi)), a, b))
        else:
            gates.append(COUPLERS[int(rng.integers(0, 6))](a, b))
    return Circuit(n, tuple(gates))


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("tile,low", [(6, 2), (9, 3), (11, 5)])
def test_lean_opcodes_vs_oracle(rng, dtype, tile, low):
    n = 14
    for seed in range(3):
        c = coupler_circuit(n, 120, 100 + seed)
        x = random_state(n, rng)
        want = O.dense_run(c.gates, x.copy(), gate_matrix)
        t = min(tile, fusion.GEOMETRY[dtype]["tile"])
        prog = compile_circuit(c, dtype=dtype, tile_bits=t, low_bits=min(low, t))
        s = DenseKet(n, x, dtype=dtype)
        prog.run(s)
        got = permute_qubits(s, prog.plan.order).amps
        assert np.max(np.abs(got - want)) < TOL[dtype], (seed, tile, low)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_couplers_only_vs_oracle(rng, dtype):
    """Pure Pauli couplers (no dense gates in between): long runs of swaps,
    Y swaps and sign flips inside one stage."""
    n = 13
    r = np.random.default_rng(7)
    gates = []
    for _ in range(200):
        a, b = (int(v) for v in r.choice(n, 2, replace=False))
        gates.append(COUPLERS[int(r.integers(0, 6))](a, b))
    c = Circuit(n, tuple(gates))
    x = random_state(n, rng)
    want = O.dense_run(c.gates, x.copy(), gate_matrix)
    prog = compile_circuit(c, dtype=dtype)
    s = DenseKet(n, x, dtype=dtype)
    prog.run(s)
    got = permute_qubits(s, prog.plan.order).amps
    assert np.max(np.abs(got - want)) < TOL[dtype]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_sweep_beyond_param_table_vs_oracle(rng, dtype):
    """A sweep with more ops than the LEAN parameter table holds (kLeanOps =
    128) runs through the generic interpreter; same results."""
    n = 8
    r = np.random.default_rng(9)
    gates = []
    for _ in range(300):  # every gate on qubits 0..2: the ops pile into few stages of one sweep
        a, b = (int(v) for v in r.choice(3, 2, replace=False))
        gates.append(u3(*r.uniform(0, 2 * math.pi, 3), a) if r.random() < 0.5 else COUPLERS[int(r.integers(0, 6))](a, b))
    c = Circuit(n, tuple(gates))
    plan = fusion.plan_circuit(c, dtype=dtype, tile_bits=8, low_bits=2)
    assert max(sum(len(st.ops) for st in sp.stages) for sp in plan.sweeps) > 128
    x = random_state(n, rng)
    want = O.dense_run(c.gates, x.copy(), gate_matrix)
    prog = compile_circuit(c, dtype=dtype, tile_bits=8, low_bits=2)
    s = DenseKet(n, x, dtype=dtype)
    prog.run(s)
    got = permute_qubits(s, prog.plan.order).amps
    assert np.max(np.abs(got - want)) < TOL[dtype]
