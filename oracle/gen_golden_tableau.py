"""Generate tests/golden/tableau.npz: the REFERENCE engine with its default
flags (stabilizer_hybrid=True) on Clifford-heavy circuits, so the native
engine's tableau shards (csrc/sk_tableau.h) are pinned decision for decision:
tableau merges, Clifford 1q words, controlled Paulis, control elimination by
deterministic eigenstates, random and deterministic tableau measurements
(rng.integers draws), p = 1 forced measurements (eps 0.5), conversions to
dense shards by log replay (a T gate), sampling and measure_all.

    python oracle/gen_golden_tableau.py          (test infrastructure only)
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from shardsim import circuit as rc  # noqa: E402
from shardsim import engine as reng  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "tableau.npz"
NAMES = ["h", "x", "y", "z", "rz", "p", "u3", "swap", "m"]
STATS = ("label_swaps", "kernels", "eliminated_controls", "merges", "splits")


def clifford_circuit(w: int, n_gates: int, seed: int, t_prob: float, m_prob: float) -> rc.Circuit:
    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(n_gates):
        r = rng.random()
        a, b = (int(v) for v in rng.choice(w, 2, replace=False))
        if r < m_prob:
            gates.append(rc.measure(a))
        elif r < m_prob + t_prob:
            gates.append(rc.phase(math.pi / 4, a))  # T: non-Clifford, converts the shard
        else:
            k = int(rng.integers(0, 14))
            if k == 0:
                gates.append(rc.h(a))
            elif k == 1:
                gates.append(rc.x(a))
            elif k == 2:
                gates.append(rc.y(a))
            elif k == 3:
                gates.append(rc.z(a))
            elif k == 4:
                gates.append(rc.phase(math.pi / 2, a))
            elif k == 5:
                gates.append(rc.phase(-math.pi / 2, a))
            elif k == 6:
                gates.append(rc.u3(math.pi / 2, 0.0, math.pi, a))  # H up to rounding
            elif k == 7:
                gates.append(rc.swap(a, b))
            else:
                gates.append([rc.cx, rc.cy, rc.cz, rc.ax, rc.ay, rc.az][k - 8](a, b))
    return rc.Circuit(w, tuple(gates))


def encode(c):
    k = len(c.gates)
    out = np.full((k, 7), -1.0)
    for i, g in enumerate(c.gates):
        out[i, 0] = NAMES.index(g.name)
        out[i, 1:1 + len(g.targets)] = g.targets
        if g.controls:
            out[i, 3], out[i, 4] = g.controls[0], g.polarity[0]
        if g.params:
            out[i, 5] = g.params[0]
            if len(g.params) == 3:
                out[i, 5:7] = g.params[0], g.params[1]
    return out


def main():
    d = {}
    cases = []
    for i in range(8):
        w = 4 + (i % 5)
        cases.append((f"c{i}", w, 40 + 10 * i, 1000 + i, 0.0 if i < 3 else 0.04, 0.06, 0.0))
    for i in range(4):  # p = 1: tableau rounding by forced measurement (engine.py:444-450)
        cases.append((f"p1_{i}", 6, 50, 2000 + i, 0.0, 0.0, 1.0))
    for i in range(3):  # p = 0.6 with T gates: tableau -> dense conversions, then SDRP on dense shards
        cases.append((f"mix{i}", 7, 60, 3000 + i, 0.08, 0.03, 0.6))
    for name, w, n_gates, seed, t_prob, m_prob, p in cases:
        c = clifford_circuit(w, n_gates, seed, t_prob, m_prob)
        sim = reng.HybridState(w, reng.EngineConfig(sdrp=p, rng_seed=seed, mem_budget=1 << 16))
        sim.apply_circuit(c)
        key = f"t/{name}"
        d[f"{key}/spec"] = np.array([w, seed], dtype=np.int64)
        d[f"{key}/p"] = p
        d[f"{key}/gates"] = encode(c)
        d[f"{key}/eps"] = np.array(sim.eps_record, dtype=float)
        d[f"{key}/stats"] = np.array([sim.stats[s] for s in STATS])
        d[f"{key}/peak"] = sim.peak_amplitudes
        d[f"{key}/kinds"] = np.array([1 if h.shard.kind == "stab" else 0 for h in sim._handles])
        d[f"{key}/ket"] = sim.full_ket().amps
        d[f"{key}/samples"] = np.array([int(s[::-1], 2) for s in sim.sample(64)], dtype=np.int64)
        d[f"{key}/measure_all"] = np.array([int(sim.measure_all()[::-1], 2)])
        d[f"{key}/ket_after"] = sim.full_ket().amps
        print(name, w, len(c.gates), "eps", len(sim.eps_record), "stats", sim.stats,
              "stab", int(d[f"{key}/kinds"].sum()))
    np.savez_compressed(OUT, **d)
    print(OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
