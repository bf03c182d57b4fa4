"""Hybrid engine over the device ket engine vs the reference engine's own
records (tests/golden/engine.npz, made by oracle/gen_golden.py): identical
SDRP decisions (eps records within 1e-9), budget peaks and OOM points,
kernel/merge/split counts, final amplitudes, measurement outcomes and
samples (same PCG64 draws).  Needs a GPU."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2304_14969_b200.circuit import Circuit, build_ghz, build_qft, build_random_circuit, measure
from paper_2304_14969_b200.engine import EngineConfig, HybridState, OptFlags
from paper_2304_14969_b200.errors import MemoryBudgetError
from paper_2304_14969_b200.sdrp import min_sdrp_search, run_hybrid

pytestmark = pytest.mark.gpu
STATS = ("label_swaps", "kernels", "eliminated_controls", "merges", "splits")


def _cases(g):
    return sorted({k.rsplit("/", 1)[0] for k in g.files if k.startswith("eng/")})


@pytest.fixture(scope="module")
def eg(golden):
    return golden("engine")


def test_engine_runs_match_reference(eg):
    for key in _cases(eg):
        w, dep, seed, budget = (int(v) for v in eg[f"{key}/spec"])
        p = float(eg[f"{key}/p"])
        fl = OptFlags(*[bool(b) for b in eg[f"{key}/flags"]])
        cfg = EngineConfig(sdrp=p, mem_budget=budget, rng_seed=seed, optimizations=fl)
        c = build_random_circuit(w, dep, seed)
        if not bool(eg[f"{key}/ok"]) and f"{key}/peak" not in eg.files:  # OOM inside the run
            with pytest.raises(MemoryBudgetError) as exc:
                sim = run_hybrid(c, cfg)
                sim.flush_all()
            assert exc.value.needed == int(eg[f"{key}/needed"]), key
            continue
        sim = run_hybrid(c, cfg)
        sim.flush_all()
        if not bool(eg[f"{key}/ok"]):  # the run fits; the 2^w readout does not (gen_golden.py records both)
            assert sim.peak_amplitudes == int(eg[f"{key}/peak"]), key
            np.testing.assert_allclose(sim.eps_record, eg[f"{key}/eps"], atol=1e-9, err_msg=key)
            with pytest.raises(MemoryBudgetError) as exc:
                sim.full_ket()
            assert exc.value.needed == int(eg[f"{key}/needed"]), key
            continue
        want = eg[f"{key}/eps"]
        assert len(sim.eps_record) == len(want), key
        np.testing.assert_allclose(sim.eps_record, want, atol=1e-9, err_msg=key)
        assert abs(sim.estimated_fidelity() - float(eg[f"{key}/fmodel"])) < 1e-9, key
        assert sim.peak_amplitudes == int(eg[f"{key}/peak"]), key
        assert [sim.stats[s] for s in STATS] == [int(v) for v in eg[f"{key}/stats"]], key  # incl. tableau runs
        got = sim.full_ket().amps
        assert np.max(np.abs(got - eg[f"{key}/ket"])) < 1e-10, key


def test_engine_qft_on_ghz(eg):
    for n in (6, 9):
        sim = HybridState(n, EngineConfig(mem_budget=1 << 20, optimizations=OptFlags(stabilizer_hybrid=False)))
        sim.apply_circuit(build_ghz(n))
        sim.apply_circuit(build_qft(n))
        assert np.max(np.abs(sim.full_ket().amps - eg[f"engqft/{n}/ket"])) < 1e-12
        assert [sim.stats[s] for s in STATS] == [int(v) for v in eg[f"engqft/{n}/stats"]]


def test_measurement_collapse_and_sampling(eg):
    for i in range(3):
        w, seed = (int(v) for v in eg[f"meas/{i}/spec"])
        c = build_random_circuit(w, 5, seed)
        gates = list(c.gates)
        gates.insert(len(gates) // 2, measure(2))
        sim = HybridState(w, EngineConfig(rng_seed=seed, optimizations=OptFlags(stabilizer_hybrid=False)))
        sim.apply_circuit(Circuit(w, tuple(gates)))
        samples = np.array([int(b[::-1], 2) for b in sim.sample(300)])
        assert np.array_equal(samples, eg[f"meas/{i}/samples"])
        assert int(sim.measure_all()[::-1], 2) == int(eg[f"meas/{i}/measure_all"][0])


def test_min_sdrp_search_matches_reference(eg):
    for key in sorted({k.rsplit("/", 1)[0] for k in eg.files if k.startswith("minsdrp/")}):
        w, dep, seed, budget = (int(v) for v in eg[f"{key}/spec"])
        feasible, p_min, f_model, peak = eg[f"{key}/res"]
        r = min_sdrp_search(w, dep, seed, budget)
        assert r.feasible == bool(feasible), key
        assert abs(r.p_min - p_min) < 1e-12 and r.peak_amplitudes == int(peak), key
        assert abs(r.f_model - f_model) <= 1e-9 * max(1.0, abs(f_model)) + 1e-15, key


def test_sdrp_round_api_and_errors():
    sim = HybridState(3, EngineConfig(optimizations=OptFlags(stabilizer_hybrid=False)))
    with pytest.raises(ValueError):
        sim.sdrp_round(0)  # width-1 shard
    from paper_2304_14969_b200.circuit import cx, h
    sim.apply_circuit(Circuit(3, (h(0), cx(0, 1))))
    sim.flush_all()
    eps = sim.sdrp_round(0, p=1.0)  # Bell pair: eps = 0.5 <= p/2
    assert abs(eps - 0.5) < 1e-12 and abs(sim.estimated_fidelity() - 0.5) < 1e-12


# ---------------------------------------------------------------------------
# tableau shards (OptFlags.stabilizer_hybrid, the default): Clifford-heavy
# circuits from oracle/gen_golden_tableau.py, run by the reference engine
# ---------------------------------------------------------------------------
def _decode(w, enc):
    from paper_2304_14969_b200.circuit import Gate
    names = ["h", "x", "y", "z", "rz", "p", "u3", "swap", "m"]
    gates = []
    for row in enc:
        name = names[int(row[0])]
        if name == "swap":
            gates.append(Gate("swap", (int(row[1]), int(row[2]))))
        elif name == "m":
            gates.append(Gate("m", (int(row[1]),)))
        else:
            params = ()
            if name == "p":
                params = (float(row[5]),)
            elif name == "u3":
                params = (float(row[5]), float(row[6]), math.pi)
            if row[3] >= 0:
                gates.append(Gate(name, (int(row[1]),), params, controls=(int(row[3]),), polarity=(int(row[4]),)))
            else:
                gates.append(Gate(name, (int(row[1]),), params))
    return Circuit(w, tuple(gates))


def test_tableau_shards_match_reference(golden):
    tg = golden("tableau")
    cases = sorted({k.split("/")[1] for k in tg.files if k.startswith("t/")})
    assert len(cases) == 15
    for name in cases:
        key = f"t/{name}"
        w, seed = (int(v) for v in tg[f"{key}/spec"])
        c = _decode(w, tg[f"{key}/gates"])
        sim = HybridState(w, EngineConfig(sdrp=float(tg[f"{key}/p"]), rng_seed=seed, mem_budget=1 << 16))
        sim.apply_circuit(c)
        np.testing.assert_allclose(sim.eps_record, tg[f"{key}/eps"], atol=1e-9, err_msg=name)
        assert [sim.stats[s] for s in STATS] == [int(v) for v in tg[f"{key}/stats"]], name
        assert sim.peak_amplitudes == int(tg[f"{key}/peak"]), name
        assert np.max(np.abs(sim.full_ket().amps - tg[f"{key}/ket"])) < 1e-10, name
        samples = np.array([int(s[::-1], 2) for s in sim.sample(64)])
        assert np.array_equal(samples, tg[f"{key}/samples"]), name
        assert int(sim.measure_all()[::-1], 2) == int(tg[f"{key}/measure_all"][0]), name
        assert np.max(np.abs(sim.full_ket().amps - tg[f"{key}/ket_after"])) < 1e-10, name
