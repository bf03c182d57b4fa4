"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run here (the only place /root/reference exists):
    python oracle/gen_golden.py
It imports shardsim from /root/reference/pkg/src (read-only; no bytecode is
written there) and records inputs and outputs of the hot-path functions, so
the oracle restatement (oracle/ket_oracle.py), the circuit builders
(paper_2304_14969_b200/circuit.py) and the GPU kernels can be checked
against the reference on machines where it is absent.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import shardsim  # noqa: E402
from shardsim import circuit as rc  # noqa: E402
from shardsim import engine as reng  # noqa: E402
from shardsim import ket as rk  # noqa: E402
from shardsim import validate as rv  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
NAMES = ["h", "x", "y", "z", "rz", "p", "u3", "swap", "m"]


def random_state(width, rng):  # conftest.py:8-10
    v = rng.normal(size=1 << width) + 1j * rng.normal(size=1 << width)
    return v / np.linalg.norm(v)


def random_unitary(rng):  # conftest.py:13-16
    z = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def encode(c):
    k = len(c.gates)
    code = np.array([NAMES.index(g.name) for g in c.gates], dtype=np.int8)
    tg = np.full((k, 2), -1, np.int16)
    ct = np.full((k, 2), -1, np.int16)
    po = np.full((k, 2), -1, np.int8)
    pa = np.zeros((k, 3))
    for i, g in enumerate(c.gates):
        tg[i, :len(g.targets)] = g.targets
        ct[i, :len(g.controls)] = g.controls
        po[i, :len(g.polarity)] = g.polarity
        pa[i, :len(g.params)] = g.params
    return dict(code=code, targets=tg, controls=ct, polarity=po, params=pa, width=np.int32(c.width))


def gen_circuits():
    d = {}
    cases = {"qft1": rc.build_qft(1), "qft2": rc.build_qft(2), "qft5": rc.build_qft(5),
             "qft20": rc.build_qft(20), "qft27": rc.build_qft(27), "ghz5": rc.build_ghz(5),
             "rand_6_4_8": rc.build_random_circuit(6, 4, 8),
             "rand_30_20_1": rc.build_random_circuit(30, 20, 1),
             "rand_30_20_d0": rc.build_random_circuit(30, 20, rv.derive_seed(0, 0)),
             "rand_54_7_d0": rc.build_random_circuit(54, 7, rv.derive_seed(0, 0)),
             "rand_54_10_d3": rc.build_random_circuit(54, 10, rv.derive_seed(0, 3)),
             "rand_17_9_5": rc.build_random_circuit(17, 9, 5)}
    for name, c in cases.items():
        for k, v in encode(c).items():
            d[f"{name}/{k}"] = v
    d["derive_seed"] = np.array([rv.derive_seed(0, i) for i in range(8)] + [rv.derive_seed(31, 2), rv.derive_seed(7, 3, 4)],
                                dtype=np.uint64)
    for name in ("h", "x", "y", "z"):
        d[f"mat/{name}"] = rc.gate_matrix(name)
    d["mat/rz"] = rc.gate_matrix("rz", (0.37,))
    d["mat/p"] = rc.gate_matrix("p", (1.1,))
    d["mat/u3"] = rc.gate_matrix("u3", (0.3, 1.7, -2.2))
    np.savez_compressed(OUT / "circuits.npz", **d)


def gen_ket():
    rng = np.random.default_rng(20240817)
    d = {}
    # apply_1q (test_ket.py:41-49 style)
    for i in range(12):
        w = int(rng.integers(1, 7))
        a = random_state(w, rng)
        q = int(rng.integers(w))
        m = random_unitary(rng) if i % 4 else rk.np.diag(np.exp(1j * rng.uniform(0, 6.28, 2)))
        s = rk.DenseKet.from_amplitudes(a)
        s.apply_1q(q, m)
        d.update({f"1q/{i}/in": a, f"1q/{i}/q": q, f"1q/{i}/m": m, f"1q/{i}/out": s.amps})
    # apply_controlled (test_ket.py:72-86 style)
    for i in range(16):
        w = int(rng.integers(2, 7))
        a = random_state(w, rng)
        qs = list(rng.permutation(w))
        nc = int(rng.integers(1, min(w, 3)))
        ctl = tuple(int(x) for x in qs[:nc])
        t = int(qs[nc])
        pol = tuple(int(b) for b in rng.integers(0, 2, nc))
        m = random_unitary(rng) if i % 3 else rc.gate_matrix("p", (float(rng.uniform(0, 6)),))
        s = rk.DenseKet.from_amplitudes(a)
        s.apply_controlled(ctl, pol, t, m)
        d.update({f"ctl/{i}/in": a, f"ctl/{i}/controls": np.array(ctl), f"ctl/{i}/polarity": np.array(pol),
                  f"ctl/{i}/target": t, f"ctl/{i}/m": m, f"ctl/{i}/out": s.amps})
    # pauli layer (test_ket.py:104-116 style)
    for i in range(10):
        w = 4
        a = random_state(w, rng)
        qubits = rng.permutation(w)[: int(rng.integers(1, w + 1))]
        layer = [(int(q), "xyz"[rng.integers(3)]) for q in qubits]
        s = rk.DenseKet.from_amplitudes(a)
        s.apply_pauli_layer(layer)
        d.update({f"pauli/{i}/in": a, f"pauli/{i}/qubits": np.array([q for q, _ in layer]),
                  f"pauli/{i}/kinds": np.array(["xyz".index(p) for _, p in layer]), f"pauli/{i}/out": s.amps})
    # bloch / probability / projection
    for i in range(10):
        w = int(rng.integers(1, 7))
        a = random_state(w, rng)
        q = int(rng.integers(w))
        s = rk.DenseKet.from_amplitudes(a)
        r = s.bloch_vector(q)
        p1 = s.probability(q, 1)
        s2 = rk.DenseKet.from_amplitudes(a)
        pr = s2.project_and_renormalize(q, 1)
        d.update({f"bloch/{i}/in": a, f"bloch/{i}/q": q, f"bloch/{i}/r": np.array([r.rx, r.ry, r.rz]),
                  f"bloch/{i}/eps": rk.epsilon_from_bloch(r), f"bloch/{i}/p1": p1, f"bloch/{i}/proj_p": pr,
                  f"bloch/{i}/proj_out": s2.amps})
    # compose / decompose / remove / permute / fidelity
    for i in range(8):
        a = random_state(1 + i % 2, rng)
        b = random_state(2 + i % 3, rng)
        ka, kb = rk.DenseKet.from_amplitudes(a), rk.DenseKet.from_amplitudes(b)
        k = ka.kron_compose(kb)
        q = int(rng.integers(k.width))
        res = k.try_decompose(q, 1e-12)
        d.update({f"kron/{i}/lo": a, f"kron/{i}/hi": b, f"kron/{i}/out": k.amps, f"kron/{i}/q": q,
                  f"kron/{i}/dec_ok": res is not None})
        if res is not None:
            d[f"kron/{i}/phi"] = res[0].amps
            d[f"kron/{i}/rest"] = res[1].amps
        order = [int(x) for x in rng.permutation(k.width)]
        d[f"kron/{i}/order"] = np.array(order)
        d[f"kron/{i}/perm"] = rk.permute_qubits(k, order).amps
        other = random_state(k.width, rng)
        d[f"kron/{i}/other"] = other
        d[f"kron/{i}/fid"] = k.fidelity(rk.DenseKet.from_amplitudes(other))
    # known-epsilon tolerance case (test_ket.py:211-218)
    a = random_state(2, rng)
    perp = random_state(2, rng)
    perp -= np.vdot(a, perp) * a
    perp /= np.linalg.norm(perp)
    amps = math.sqrt(0.999) * np.kron(a, [1, 0]) + math.sqrt(0.001) * np.kron(perp, [0, 1])
    d["eps_case/in"] = amps
    d["eps_case/dec_1e-6"] = rk.DenseKet.from_amplitudes(amps).try_decompose(0, 1e-6) is not None
    r3 = rk.DenseKet.from_amplitudes(amps).try_decompose(0, 1e-3)
    d["eps_case/phi"] = r3[0].amps
    d["eps_case/rest"] = r3[1].amps
    # remove_qubit on a product with |0>
    base = random_state(3, rng)
    prod = np.kron(base, [1, 0])
    d["remove/in"] = prod
    d["remove/out"] = rk.DenseKet.from_amplitudes(prod).remove_qubit(0).amps
    # measurement sampling draw-for-draw (engine.py:613-615, 648-650)
    for i in range(4):
        w = 3 + 2 * i
        a = random_state(w, rng)
        g = np.random.default_rng(100 + i)
        probs = np.abs(a) ** 2
        probs /= probs.sum()
        draws = g.choice(probs.size, size=257, p=probs)
        g2 = np.random.default_rng(100 + i)
        d.update({f"sample/{i}/in": a, f"sample/{i}/seed": 100 + i, f"sample/{i}/draws": draws,
                  f"sample/{i}/uniforms": g2.random(257)})
    # SDRP rounding step (engine.py:464-488) via the engine's own method
    for i in range(6):
        w = 3 + i % 3
        a = random_state(w, rng)
        q = int(rng.integers(w))
        sim = reng.HybridState(w, reng.EngineConfig(sdrp=1.0, optimizations=reng.OptFlags.none()))
        sim.load_state(rk.DenseKet.from_amplitudes(a))
        sh = sim._handles[q].shard
        r = sh.state.bloch_vector(q)
        eps = rk.epsilon_from_bloch(r)
        rec = sim._round_qubit(sh, q, r, eps)
        d.update({f"round/{i}/in": a, f"round/{i}/q": q, f"round/{i}/eps": eps,
                  f"round/{i}/rec": -1.0 if rec is None else rec,
                  f"round/{i}/phi": sim._handles[q].shard.state.amps, f"round/{i}/rest": sh.state.amps})
    np.savez_compressed(OUT / "ket_ops.npz", **d)


def gen_qft():
    rng = np.random.default_rng(7)
    d = {}
    for n in (2, 3, 5, 8, 10, 12):
        x = random_state(n, rng)
        got = rv.dense_reference(rc.build_qft(n), initial=rk.DenseKet(n, x.copy()))
        d[f"qft/{n}/in"] = x
        d[f"qft/{n}/out"] = got.amps
        d[f"qft/{n}/dft"] = rv.dft_oracle(x)
    # GHZ input, paper Fig. 1b path, n = 16
    n = 16
    x = np.zeros(1 << n, complex)
    x[0] = x[-1] = 2 ** -0.5
    d["ghz16/out"] = rv.dense_reference(rc.build_qft(n), initial=rk.DenseKet(n, x.copy())).amps
    # exact random circuits (dense_reference from |0..0>)
    for (w, dep, seed) in ((6, 4, 8), (10, 6, 3), (14, 8, rv.derive_seed(0, 1))):
        d[f"rand/{w}_{dep}_{seed}/out"] = rv.dense_reference(rc.build_random_circuit(w, dep, seed)).amps
        d[f"rand/{w}_{dep}_{seed}/spec"] = np.array([w, dep, seed], dtype=np.uint64)
    np.savez_compressed(OUT / "qft_dense.npz", **d)


def gen_engine():
    """Reference HybridState runs (stabilizer path off and default flags) that
    the device engine must reproduce decision for decision."""
    d = {}
    none = reng.OptFlags.none()
    nostab = reng.OptFlags(stabilizer_hybrid=False)
    cases = []
    for i in range(6):
        w, dep = [(6, 4), (8, 6), (10, 8), (12, 10), (9, 12), (14, 6)][i]
        seed = rv.derive_seed(5, i)
        for p in (0.0, 0.3, 0.6, 1.0):
            for fl_name, fl in (("nostab", nostab), ("default", reng.OptFlags()), ("none", none)):
                if fl_name == "none" and p not in (0.0, 0.6):
                    continue
                cases.append((f"rc{i}_p{int(p * 10)}_{fl_name}", w, dep, seed, p, 1 << 12, fl))
    for name, w, dep, seed, p, budget, fl in cases:
        c = rc.build_random_circuit(w, dep, seed)
        cfg = reng.EngineConfig(sdrp=p, mem_budget=budget, rng_seed=seed, optimizations=fl)
        key = f"eng/{name}"
        d[f"{key}/spec"] = np.array([w, dep, seed, budget], dtype=np.uint64)
        d[f"{key}/p"] = p
        d[f"{key}/flags"] = np.array([fl.control_elimination, fl.hx_commutation, fl.label_swap,
                                      fl.pauli_coalescing, fl.stabilizer_hybrid], dtype=bool)
        try:
            sim = rv.run_hybrid(c, cfg)
            sim.flush_all()
            d[f"{key}/ok"] = True
            d[f"{key}/eps"] = np.array(sim.eps_record, dtype=float)
            d[f"{key}/fmodel"] = sim.estimated_fidelity()
            d[f"{key}/peak"] = sim.peak_amplitudes
            d[f"{key}/stats"] = np.array([sim.stats[k] for k in ("label_swaps", "kernels", "eliminated_controls",
                                                                 "merges", "splits")])
            d[f"{key}/ket"] = sim.full_ket().amps
        except reng.MemoryBudgetError as exc:
            d[f"{key}/ok"] = False
            d[f"{key}/needed"] = exc.needed
    # QFT on GHZ through the engine (the paper's Fig. 1b path), n = 8
    for n in (6, 9):
        sim = reng.HybridState(n, reng.EngineConfig(mem_budget=1 << 20, optimizations=nostab))
        sim.apply_circuit(rc.build_ghz(n))
        sim.apply_circuit(rc.build_qft(n))
        d[f"engqft/{n}/ket"] = sim.full_ket().amps
        d[f"engqft/{n}/stats"] = np.array([sim.stats[k] for k in ("label_swaps", "kernels", "eliminated_controls",
                                                                  "merges", "splits")])
    # measurement, collapse and sampling with the engine rng
    for i in range(3):
        w = 7 + i
        seed = 100 + i
        c = rc.build_random_circuit(w, 5, seed)
        gates = list(c.gates)
        gates.insert(len(gates) // 2, rc.measure(2))
        cm = rc.Circuit(w, tuple(gates))
        sim = reng.HybridState(w, reng.EngineConfig(rng_seed=seed, optimizations=nostab))
        sim.apply_circuit(cm)
        d[f"meas/{i}/spec"] = np.array([w, seed], dtype=np.uint64)
        d[f"meas/{i}/samples"] = np.array([int(b[::-1], 2) for b in sim.sample(300)], dtype=np.int64)
        d[f"meas/{i}/measure_all"] = np.array([int(sim.measure_all()[::-1], 2)])
    # min-SDRP searches (validate.py:280-300), incl. 54 qubits x 7 layers
    for (w, dep, i, budget) in ((16, 6, 0, 1 << 10), (16, 8, 1, 1 << 10), (54, 7, 2, 1 << 18)):
        seed = rv.derive_seed(0, i)
        r = rv.min_sdrp_search(w, dep, seed, budget)
        d[f"minsdrp/{w}_{dep}_{i}/spec"] = np.array([w, dep, seed, budget], dtype=np.uint64)
        d[f"minsdrp/{w}_{dep}_{i}/res"] = np.array([r.feasible, -1 if r.p_min is None else r.p_min,
                                                    -1 if r.f_model is None else r.f_model, r.peak_amplitudes],
                                                   dtype=float)
        if r.feasible:
            sim = rv.run_hybrid(rc.build_random_circuit(w, dep, seed),
                                reng.EngineConfig(sdrp=r.p_min, mem_budget=budget, rng_seed=seed))
            sim.flush_all()
            d[f"minsdrp/{w}_{dep}_{i}/eps"] = np.array(sim.eps_record)
    np.savez_compressed(OUT / "engine.npz", **d)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    assert shardsim.RNG_ALGORITHM == "pcg64"
    gen_circuits()
    gen_ket()
    gen_qft()
    gen_engine()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
