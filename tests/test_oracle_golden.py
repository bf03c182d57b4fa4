"""Pin the CPU oracle to the reference: every oracle function reproduces the
outputs the reference package itself produced (tests/golden/*.npz, made by
oracle/gen_golden.py).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import ket_oracle as O
from paper_2304_14969_b200.circuit import gate_matrix


@pytest.fixture(scope="module")
def kg(golden):
    return golden("ket_ops")


def _cases(g, prefix):
    return sorted({k.split("/")[1] for k in g.files if k.startswith(prefix + "/")}, key=int)


def test_apply_1q(kg):
    for i in _cases(kg, "1q"):
        a = kg[f"1q/{i}/in"].copy()
        O.apply_1q(a, int(kg[f"1q/{i}/q"]), kg[f"1q/{i}/m"])
        assert np.array_equal(a, kg[f"1q/{i}/out"])


def test_apply_controlled(kg):
    for i in _cases(kg, "ctl"):
        a = kg[f"ctl/{i}/in"].copy()
        O.apply_controlled(a, tuple(kg[f"ctl/{i}/controls"]), tuple(kg[f"ctl/{i}/polarity"]),
                           int(kg[f"ctl/{i}/target"]), kg[f"ctl/{i}/m"])
        assert np.array_equal(a, kg[f"ctl/{i}/out"])


def test_pauli_layer(kg):
    for i in _cases(kg, "pauli"):
        layer = [(int(q), "xyz"[k]) for q, k in zip(kg[f"pauli/{i}/qubits"], kg[f"pauli/{i}/kinds"])]
        out = O.apply_pauli_layer(kg[f"pauli/{i}/in"], layer)
        assert np.array_equal(out, kg[f"pauli/{i}/out"])


def test_bloch_probability_projection(kg):
    for i in _cases(kg, "bloch"):
        a = kg[f"bloch/{i}/in"]
        q = int(kg[f"bloch/{i}/q"])
        r = O.bloch_vector(a, q)
        assert np.array_equal(np.array(r), kg[f"bloch/{i}/r"])
        assert O.epsilon(r) == float(kg[f"bloch/{i}/eps"])
        assert O.probability(a, q, 1) == float(kg[f"bloch/{i}/p1"])
        b = a.copy()
        assert O.project_and_renormalize(b, q, 1) == float(kg[f"bloch/{i}/proj_p"])
        assert np.array_equal(b, kg[f"bloch/{i}/proj_out"])


def test_compose_decompose_permute_fidelity(kg):
    for i in _cases(kg, "kron"):
        k = O.kron_compose(kg[f"kron/{i}/lo"], kg[f"kron/{i}/hi"])
        assert np.array_equal(k, kg[f"kron/{i}/out"])
        res = O.try_decompose(k, int(kg[f"kron/{i}/q"]), 1e-12)
        assert (res is not None) == bool(kg[f"kron/{i}/dec_ok"])
        if res is not None:
            assert np.array_equal(res[0], kg[f"kron/{i}/phi"])
            assert np.array_equal(res[1], kg[f"kron/{i}/rest"])
        assert np.array_equal(O.permute_qubits(k, list(kg[f"kron/{i}/order"])), kg[f"kron/{i}/perm"])
        assert O.fidelity(k, kg[f"kron/{i}/other"]) == float(kg[f"kron/{i}/fid"])


def test_known_epsilon_and_remove(kg):
    a = kg["eps_case/in"]
    assert (O.try_decompose(a, 0, 1e-6) is not None) == bool(kg["eps_case/dec_1e-6"])
    phi, rest = O.try_decompose(a, 0, 1e-3)
    assert np.array_equal(phi, kg["eps_case/phi"]) and np.array_equal(rest, kg["eps_case/rest"])
    assert np.array_equal(O.remove_qubit(kg["remove/in"], 0), kg["remove/out"])


def test_sampling_draw_for_draw(kg):
    for i in _cases(kg, "sample"):
        g = np.random.default_rng(int(kg[f"sample/{i}/seed"]))
        assert np.array_equal(O.sample(kg[f"sample/{i}/in"], g, 257), kg[f"sample/{i}/draws"])
        # the device path's contract: cumsum / normalise / searchsorted('right') on host uniforms
        a = kg[f"sample/{i}/in"]
        p = np.abs(a) ** 2
        cdf = np.cumsum(p / p.sum())
        cdf /= cdf[-1]
        idx = np.searchsorted(cdf, kg[f"sample/{i}/uniforms"], side="right")
        assert np.array_equal(idx, kg[f"sample/{i}/draws"])


def test_sdrp_round_step(kg):
    for i in _cases(kg, "round"):
        res = O.round_qubit(kg[f"round/{i}/in"], int(kg[f"round/{i}/q"]))
        assert res is not None
        phi, rest = res
        np.testing.assert_allclose(phi, kg[f"round/{i}/phi"], atol=1e-15)
        np.testing.assert_allclose(rest, kg[f"round/{i}/rest"], atol=1e-15)


def test_qft_dense_loop_and_dft(golden):
    g = golden("qft_dense")
    from paper_2304_14969_b200.circuit import build_qft
    for n in (2, 3, 5, 8, 10, 12):
        x = g[f"qft/{n}/in"]
        out = O.dense_run(build_qft(n).gates, x.copy(), gate_matrix)
        assert np.array_equal(out, g[f"qft/{n}/out"])
        assert np.array_equal(O.dft_oracle(x), g[f"qft/{n}/dft"])
        # label-swap variant (engine.py:525-535) equals the SWAP-kernel result after relabelling
        ls = O.dense_run(build_qft(n).gates, x.copy(), gate_matrix, label_swap=True)
        phys = O.swap_permutation(build_qft(n).gates, n)
        assert np.max(np.abs(O.permute_qubits(ls, phys) - g[f"qft/{n}/out"])) < 1e-14
    n = 16
    ghz = g["ghz16/out"]
    assert np.max(np.abs(O.qft_of_ghz(n, np.arange(1 << n)) - ghz)) < 1e-13
    x = np.zeros(1 << n, complex)
    x[0] = x[-1] = 2 ** -0.5
    np.testing.assert_allclose(O.dft_at(x, [0, 1, 5, 40000]), ghz[[0, 1, 5, 40000]], atol=1e-13)


def test_random_circuits_dense(golden):
    g = golden("qft_dense")
    from paper_2304_14969_b200.circuit import build_random_circuit
    for key in [k for k in g.files if k.startswith("rand/") and k.endswith("/spec")]:
        w, d, s = (int(v) for v in g[key])
        x = np.zeros(1 << w, complex)
        x[0] = 1
        out = O.dense_run(build_random_circuit(w, d, s).gates, x, gate_matrix)
        assert np.array_equal(out, g[key.replace("/spec", "/out")])


def test_reference_engine_stabilizer_path_is_decision_neutral_on_random_circuits(golden):
    """Recorded fact backing the dense-only engine: on the random-circuit
    workloads the reference engine makes the same SDRP decisions (eps record,
    peak, OOM point) with and without its stabilizer path."""
    g = golden("engine")
    keys = sorted({k.rsplit("/", 1)[0] for k in g.files if k.startswith("eng/")})
    keys = [k for k in keys if k.endswith("_nostab")]
    assert len(keys) >= 20
    for k in keys:
        k2 = k.replace("_nostab", "_default")
        assert bool(g[k + "/ok"]) == bool(g[k2 + "/ok"])
        if bool(g[k + "/ok"]):
            assert np.array_equal(g[k + "/eps"], g[k2 + "/eps"])
            assert int(g[k + "/peak"]) == int(g[k2 + "/peak"])
        else:
            assert int(g[k + "/needed"]) == int(g[k2 + "/needed"])
