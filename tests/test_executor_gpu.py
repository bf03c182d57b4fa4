"""Fused dense executor parity on the GPU.

Small sizes: bit-for-bit-level agreement (1e-12 fp64 / 1e-5 fp32 per element,
north_star's tolerances) with the oracle's gate-by-gate dense loop and with
the reference's own golden outputs.  Full sizes (27 qubits): closed forms
that need no CPU oracle — the QFT of GHZ (y_j = (1 + e^{-2 pi i j/N})/sqrt(2N))
and of a basis state |k> (y_j = e^{2 pi i jk/N}/sqrt(N)) — plus norm."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import ket_oracle as O
from paper_2304_14969_b200 import fusion
from paper_2304_14969_b200.circuit import (Circuit, build_ghz, build_qft, build_random_circuit, cp, cx, gate_matrix,
                                           h, measure, rz, swap, u3)
from paper_2304_14969_b200.executor import Program, compile_circuit, dense_reference
from paper_2304_14969_b200.ket import DenseKet

from conftest import random_state

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 1e-5}


@pytest.mark.parametrize("n", [10, 13, 16])
def test_qft_five_register_bits_vs_oracle(rng, n):
    x = random_state(n, rng)
    prog = compile_circuit(build_qft(n), dtype="c64", tile_bits=min(n, 13), low_bits=4, qft_nreg=5)
    assert prog.plan.nreg == 5
    s = DenseKet(n, x, dtype="c64")
    prog.run(s)
    from paper_2304_14969_b200.ket import permute_qubits
    got = permute_qubits(s, prog.plan.order).amps
    assert np.max(np.abs(got - O.dft_oracle(x))) < 1e-5


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_qft_small_vs_oracle_and_dft(rng, dtype):
    for n in range(2, 15):
        for _ in range(3 if n < 12 else 1):
            x = random_state(n, rng)
            got = dense_reference(build_qft(n), initial=DenseKet(n, x, dtype=dtype)).amps
            want = O.dense_run(build_qft(n).gates, x.copy(), gate_matrix)
            assert np.max(np.abs(got - want)) < TOL[dtype], n
            assert np.max(np.abs(got - O.dft_oracle(x))) < TOL[dtype], n


def test_qft_golden_from_reference(golden):
    g = golden("qft_dense")
    for n in (2, 3, 5, 8, 10, 12):
        got = dense_reference(build_qft(n), initial=DenseKet(n, g[f"qft/{n}/in"])).amps
        assert np.max(np.abs(got - g[f"qft/{n}/out"])) < 1e-12
    n = 16
    x = np.zeros(1 << n, complex)
    x[0] = x[-1] = 2 ** -0.5
    got = dense_reference(build_qft(n), initial=DenseKet(n, x)).amps
    assert np.max(np.abs(got - g["ghz16/out"])) < 1e-12


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_random_circuits_golden(golden, dtype):
    g = golden("qft_dense")
    for key in [k for k in g.files if k.startswith("rand/") and k.endswith("/spec")]:
        w, d, s = (int(v) for v in g[key])
        got = dense_reference(build_random_circuit(w, d, s), dtype=dtype).amps
        assert np.max(np.abs(got - g[key.replace("/spec", "/out")])) < TOL[dtype], key


@pytest.mark.parametrize("tile,low", [(6, 2), (8, 0), (10, 5), (13, 5)])
def test_plan_geometries(rng, tile, low):
    """Same circuit through different tile/low-bit geometries (exercises the
    deposit, swizzle, stage exchanges and edge-stage padding)."""
    n = 15
    c = build_random_circuit(n, 5, 11)
    x = random_state(n, rng)
    want = O.dense_run(c.gates, x.copy(), gate_matrix)
    for dtype in ("c128", "c64"):
        geo_tile = min(tile, fusion.GEOMETRY[dtype]["tile"])
        prog = compile_circuit(c, dtype=dtype, tile_bits=geo_tile, low_bits=min(low, geo_tile))
        s = DenseKet(n, x, dtype=dtype)
        prog.run(s)
        from paper_2304_14969_b200.ket import permute_qubits
        got = permute_qubits(s, prog.plan.order).amps
        assert np.max(np.abs(got - want)) < TOL[dtype]


def test_mixed_controls_swaps_and_measurement(rng):
    n = 14
    from paper_2304_14969_b200.circuit import Gate
    gates = [h(0), cx(0, 13), swap(1, 12), u3(0.3, 0.2, 0.1, 12), rz(0.4, 3), cp(0.7, 3, 11),
             Gate("y", (5,), controls=(2, 9), polarity=(1, 0)), swap(0, 8), cx(8, 2), h(4)]
    gates += [cp(math.pi / (1 << k), 6 - k, 6) for k in range(1, 7)]
    c = Circuit(n, tuple(gates))
    x = random_state(n, rng)
    got = dense_reference(c, initial=DenseKet(n, x)).amps
    want = O.dense_run(c.gates, x.copy(), gate_matrix)
    assert np.max(np.abs(got - want)) < 1e-12
    cm = Circuit(n, tuple(gates[:5]) + (measure(3),) + tuple(gates[5:]) + (measure(12),))
    got = dense_reference(cm, initial=DenseKet(n, x), rng=np.random.default_rng(3)).amps
    want = O.dense_run(cm.gates, x.copy(), gate_matrix, rng=np.random.default_rng(3))
    assert np.max(np.abs(got - want)) < 1e-12
    with pytest.raises(ValueError):
        dense_reference(cm, initial=DenseKet(n, x))


@pytest.mark.parametrize("dtype,qft_nreg", [("c64", None), ("c128", None), ("c64", 5)])
def test_qft27_closed_forms(dtype, qft_nreg):
    """Config D2 (27 qubits, 1xB200) checked with size-independent closed forms
    (qft_nreg=5: the 32-amplitudes-per-thread QFT-window kernel)."""
    n = 27
    N = 1 << n
    kw = dict(tile_bits=13, low_bits=4, qft_nreg=5) if qft_nreg else {}
    prog = compile_circuit(build_qft(n), dtype=dtype, **kw)
    assert prog.n_sweeps == 3
    idx = np.random.default_rng(1).integers(0, N, 4096)
    from paper_2304_14969_b200.ket import permute_qubits
    # GHZ input (paper Fig. 1b)
    x = np.zeros(N, complex)
    x[0] = x[-1] = 2 ** -0.5
    s = DenseKet(n, x, dtype=dtype)
    prog.run(s)
    out = permute_qubits(s, prog.plan.order)
    amps = out.amps
    tol = 2e-15 if dtype == "c128" else 2e-9  # |y_j| <= 1.2e-4: relative 1e-11 (fp64) / 2e-5 (fp32)
    assert np.max(np.abs(amps[idx] - O.qft_of_ghz(n, idx))) < tol
    assert np.max(np.abs(amps - O.qft_of_ghz(n, np.arange(N)))) < tol
    assert abs(out.norm() - 1) < (1e-12 if dtype == "c128" else 1e-5)
    del amps, out
    # basis-state input |k>: y_j = exp(2 pi i j k / N) / sqrt(N)
    k = 0x5A5A5A5 % N
    x = np.zeros(N, complex)
    x[k] = 1
    s = DenseKet(n, x, dtype=dtype)
    prog.run(s)
    amps = permute_qubits(s, prog.plan.order).amps
    want = np.exp(2j * np.pi * ((np.arange(N, dtype=np.int64) * k) % N) / N) / math.sqrt(N)
    assert np.max(np.abs(amps - want)) < (1e-15 if dtype == "c128" else 2e-9)


@pytest.mark.parametrize("world,n_local", [(2, 9), (4, 11), (8, 13)])
def test_sharded_qft_plans_on_device(world, n_local):
    """The per-rank device programs of the global-qubit sharded QFT (rank-
    dependent top-layer sweep + local QFT body) run through the real kernels
    on one GPU, with the all-to-all block exchange done on the host."""
    from paper_2304_14969_b200 import distributed as D
    n, G = D.layout(n_local, world)
    rng = np.random.default_rng(world)
    x = random_state(n, rng)
    slabs = [DenseKet(n_local, s, dtype="c64") for s in np.split(x.copy(), world)]

    def exchange():
        host = D.exchange_blocks([k.amps for k in slabs])
        for k, h in zip(slabs, host):
            k.amps = h

    exchange()
    for r, k in enumerate(slabs):
        top, _ = D.plans(n_local, world, r, "c64")
        Program(top).run(k)
    exchange()
    for r, k in enumerate(slabs):
        _, body = D.plans(n_local, world, r, "c64")
        Program(body).run(k)
    out = np.concatenate([k.amps for k in slabs])
    got = O.permute_qubits(out, D.final_order(n))
    assert np.max(np.abs(got - O.dft_oracle(x))) < 1e-5


def test_phase_index_offset_validation():
    """sk_program_set_phase_index: QFT-window programs only; value < 2^shift."""
    from paper_2304_14969_b200 import fusion
    prog = Program(fusion.plan_qft(12, "c64"))
    with pytest.raises(ValueError):
        prog.set_phase_index(2, 4)  # value needs more than 2 bits
    prog.set_phase_index(2, 3)
    prog.set_phase_index(0, 0)
    gen = compile_circuit(build_random_circuit(12, 3, 1), dtype="c64")
    with pytest.raises(ValueError):
        gen.set_phase_index(1, 1)  # generic sweeps cannot fold rank-constant phases
