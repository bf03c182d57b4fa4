"""The package's circuit builders emit exactly the reference's circuits
(tests/golden/circuits.npz from the reference's own builders).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2304_14969_b200 import circuit as C

NAMES = ["h", "x", "y", "z", "rz", "p", "u3", "swap", "m"]
CASES = {"qft1": lambda: C.build_qft(1), "qft2": lambda: C.build_qft(2), "qft5": lambda: C.build_qft(5),
         "qft20": lambda: C.build_qft(20), "qft27": lambda: C.build_qft(27), "ghz5": lambda: C.build_ghz(5),
         "rand_6_4_8": lambda: C.build_random_circuit(6, 4, 8),
         "rand_30_20_1": lambda: C.build_random_circuit(30, 20, 1),
         "rand_30_20_d0": lambda: C.build_random_circuit(30, 20, C.derive_seed(0, 0)),
         "rand_54_7_d0": lambda: C.build_random_circuit(54, 7, C.derive_seed(0, 0)),
         "rand_54_10_d3": lambda: C.build_random_circuit(54, 10, C.derive_seed(0, 3)),
         "rand_17_9_5": lambda: C.build_random_circuit(17, 9, 5)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_builder_matches_reference(golden, name):
    g = golden("circuits")
    c = CASES[name]()
    assert c.width == int(g[f"{name}/width"])
    code = g[f"{name}/code"]
    assert len(c.gates) == len(code)
    for i, gate in enumerate(c.gates):
        assert gate.name == NAMES[code[i]]
        tg = [int(v) for v in g[f"{name}/targets"][i] if v >= 0]
        ct = [int(v) for v in g[f"{name}/controls"][i] if v >= 0]
        po = [int(v) for v in g[f"{name}/polarity"][i] if v >= 0]
        assert list(gate.targets) == tg and list(gate.controls) == ct and list(gate.polarity) == po
        pa = g[f"{name}/params"][i][: len(gate.params)]
        assert tuple(gate.params) == tuple(float(v) for v in pa)  # bit-exact angles


def test_gate_matrices_and_seeds(golden):
    g = golden("circuits")
    for name in ("h", "x", "y", "z"):
        assert np.array_equal(C.gate_matrix(name), g[f"mat/{name}"])
    assert np.array_equal(C.gate_matrix("rz", (0.37,)), g["mat/rz"])
    assert np.array_equal(C.gate_matrix("p", (1.1,)), g["mat/p"])
    assert np.array_equal(C.gate_matrix("u3", (0.3, 1.7, -2.2)), g["mat/u3"])
    seeds = [C.derive_seed(0, i) for i in range(8)] + [C.derive_seed(31, 2), C.derive_seed(7, 3, 4)]
    assert np.array_equal(np.array(seeds, dtype=np.uint64), g["derive_seed"])


def test_gate_validation():
    with pytest.raises(ValueError):
        C.Gate("h", (0, 1))
    with pytest.raises(ValueError):
        C.Gate("x", (0,), controls=(0,), polarity=(1,))
    with pytest.raises(ValueError):
        C.Gate("swap", (0, 1), controls=(2,), polarity=(1,))
    with pytest.raises(ValueError):
        C.Circuit(2, (C.h(2),))
    with pytest.raises(ValueError):
        C.build_random_circuit(1, 3, 0)
