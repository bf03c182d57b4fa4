"""B200-native dense ket engine: a drop-in for shardsim's `DenseKet` hot path.

Reference: arXiv 2304.14969 (Qrack) as re-created by the `shardsim` package.
The amplitudes live in HBM and every kernel is hand-written sm_100a CUDA in
libshardcu.so (C ABI: include/shardcu.h).  There is no CPU fallback.
"""
from .circuit import (Circuit, Gate, build_ghz, build_qft, build_random_circuit, derive_seed,
                      gate_matrix, u3_matrix)
from .errors import DeviceError, InvariantError, MemoryBudgetError
from .ket import BlochVector, DenseKet, bloch_to_state, epsilon_from_bloch, permute_qubits

__version__ = "0.1.0"
RNG_ALGORITHM = "pcg64"

__all__ = [
    "BlochVector", "Circuit", "DenseKet", "DeviceError", "Gate", "InvariantError", "MemoryBudgetError",
    "bloch_to_state", "build_ghz", "build_qft", "build_random_circuit", "derive_seed", "epsilon_from_bloch",
    "gate_matrix", "permute_qubits", "u3_matrix",
]
