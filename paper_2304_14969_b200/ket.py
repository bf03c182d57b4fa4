"""Device-resident dense shards: the drop-in for the reference's `DenseKet`.

Mirrors `pkg/src/shardsim/ket.py` (the reference's hot path) method for
method — same names, argument meaning, exceptions and instrumentation
counters — with the amplitudes living in B200 HBM and every kernel running
in libshardcu (include/shardcu.h).  There is no CPU path: constructing a
DenseKet without a CUDA device raises.

Amplitude index convention (ket.py:3-4): qubit 0 is the least-significant
bit of the basis-state index.

`.amps` is a host *snapshot*: reading it downloads the state; assigning to
it (including `ket.amps *= z`, which Python lowers to get + set) uploads.
Item assignment into a downloaded array does not write through.

Extra device-native methods the hybrid engine uses (not in the reference):
`apply_controlled_bloch` (gate + both operand Bloch vectors in one pass),
`round_qubit` (fused SDRP rotate-project-compact), `split_measured`,
`scale`, `swap_qubits`, `sample_indices`.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import call

alloc_count = 0       # ket.py:19 — DenseKet constructions
amplitude_writes = 0  # ket.py:20 — amplitudes written by mutating kernels

_UNITARY_TOL = 1e-10  # ket.py:22

_default_dtype = "c128"  # the reference is always complex128 (ket.py:77,82)
_default_device = 0


def set_default_dtype(dtype: str) -> None:
    """'c128' (reference precision, default) or 'c64' (fp32 storage)."""
    global _default_dtype
    if dtype not in _lib.DTYPES:
        raise ValueError(f"unknown dtype {dtype!r}")
    _default_dtype = "c64" if _lib.DTYPES[dtype] == _lib.SK_C64 else "c128"


def get_default_dtype() -> str:
    return _default_dtype


def set_default_device(device: int) -> None:
    global _default_device
    _default_device = int(device)


def get_default_device() -> int:
    return _default_device


@dataclass(frozen=True)
class BlochVector:
    """Pauli expectation values (<X>, <Y>, <Z>) of one qubit (ket.py:25-34)."""

    rx: float
    ry: float
    rz: float

    def length(self) -> float:
        return math.sqrt(self.rx * self.rx + self.ry * self.ry + self.rz * self.rz)


def epsilon_from_bloch(r: BlochVector) -> float:
    """Schmidt branch weight (1 - |r|)/2 of the 1-vs-rest split (ket.py:37-39)."""
    return (1.0 - min(r.length(), 1.0)) / 2.0


def bloch_to_state(r: BlochVector) -> np.ndarray:
    """Unit Bloch vector -> pure single-qubit state along it (ket.py:42-54)."""
    norm = r.length()
    if norm < 1e-15:
        raise ValueError("zero Bloch vector has no associated pure state")
    nz = r.rz / norm
    c = math.sqrt(max(0.0, (1.0 + nz) / 2.0))
    s = math.sqrt(max(0.0, (1.0 - nz) / 2.0))
    if s < 1e-15:
        return np.array([1.0, 0.0], dtype=complex)
    a = math.atan2(r.ry / norm, r.rx / norm)
    return np.array([c, s * np.exp(1j * a)], dtype=complex)


def bloch_from_sums(sums) -> BlochVector:
    """(Re, Im of sum conj(a0) a1, sum|a0|^2, sum|a1|^2) -> Bloch vector (ket.py:204-210)."""
    cr, ci, n0, n1 = sums
    return BlochVector(2.0 * cr, 2.0 * ci, n0 - n1)


def _check_unitary(m: np.ndarray) -> None:
    if np.max(np.abs(m.conj().T @ m - np.eye(2))) > _UNITARY_TOL:
        raise ValueError("matrix is not unitary within 1e-10")


def _as_mat(m) -> np.ndarray:
    m = np.asarray(m, dtype=complex)
    if m.shape != (2, 2):
        raise ValueError(f"need a 2x2 matrix, got shape {m.shape}")
    return m


class DenseKet:
    """A ``width``-qubit shard of 2**width complex amplitudes in device memory.

    Mutating kernels never renormalise; only projections rescale (ket.py:62-66).
    Single-writer contract: one mutating operation at a time per shard.
    """

    __slots__ = ("width", "dtype", "device", "_h", "_owned", "__weakref__")

    def __init__(self, width: int, amps: np.ndarray | None = None, *, dtype: str | None = None,
                 device: int | None = None, _handle=None, _borrowed: bool = False):
        global alloc_count
        if width < 1:
            raise ValueError("shard width must be >= 1")
        self.width = width
        self.dtype = _default_dtype if dtype is None else ("c64" if _lib.DTYPES[dtype] == _lib.SK_C64 else "c128")
        self.device = _default_device if device is None else int(device)
        self._h = None
        self._owned = not _borrowed
        code = _lib.DTYPES[self.dtype]
        h = C.c_void_p()
        if _handle is not None:
            h = _handle
        elif amps is None:
            _lib.require_device()
            call("sk_create", width, code, self.device, C.byref(h), needed=1 << width)
        else:
            if amps.shape != (1 << width,):
                raise ValueError(f"need {1 << width} amplitudes, got {amps.shape}")
            _lib.require_device()
            buf = np.ascontiguousarray(amps, dtype=np.complex128)
            call("sk_create_from", width, code, self.device, buf.ctypes.data_as(_lib.dptr), C.byref(h),
                 needed=1 << width)
        self._h = h
        if not _borrowed:
            alloc_count += 1

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None and getattr(self, "_owned", True):
            try:
                _lib._lib.sk_destroy(h)
            except Exception:
                pass
            self._h = None

    def _new(self, handle, width: int) -> "DenseKet":
        return DenseKet(width, dtype=self.dtype, device=self.device, _handle=handle)

    # ------------------------------------------------------------------
    # construction / host views
    # ------------------------------------------------------------------
    @classmethod
    def from_amplitudes(cls, amps, **kw) -> "DenseKet":
        amps = np.asarray(amps, dtype=complex)
        width = int(round(math.log2(amps.size))) if amps.size else 0
        if amps.size == 0 or 1 << width != amps.size:
            raise ValueError("amplitude count must be a power of two")
        return cls(width, amps.copy(), **kw)

    def copy(self) -> "DenseKet":
        h = C.c_void_p()
        call("sk_copy", self._h, C.byref(h), needed=1 << self.width)
        return self._new(h, self.width)

    @property
    def size(self) -> int:
        return 1 << self.width

    @property
    def amps(self) -> np.ndarray:
        out = np.empty(1 << self.width, dtype=np.complex128)
        call("sk_download", self._h, out.ctypes.data_as(_lib.dptr), out.size)
        return out

    @amps.setter
    def amps(self, value) -> None:
        buf = np.ascontiguousarray(value, dtype=np.complex128)
        if buf.shape != (1 << self.width,):
            raise ValueError(f"need {1 << self.width} amplitudes, got {buf.shape}")
        call("sk_upload", self._h, buf.ctypes.data_as(_lib.dptr), buf.size)

    def device_ptr(self) -> int:
        p = C.c_uint64()
        call("sk_device_ptr", self._h, C.byref(p))
        return int(p.value)

    def norm(self) -> float:
        out = C.c_double()
        call("sk_norm2", self._h, C.byref(out))
        return math.sqrt(out.value)

    def _axis(self, q: int) -> int:
        if not 0 <= q < self.width:
            raise IndexError(f"qubit {q} out of range for width {self.width}")
        return self.width - 1 - q

    # ------------------------------------------------------------------
    # kernels
    # ------------------------------------------------------------------
    def apply_1q(self, q: int, m) -> None:
        """Apply a 2x2 unitary to qubit q (ket.py:128-131)."""
        m = _as_mat(m)
        _check_unitary(m)
        self._apply_1q_unchecked(q, m)

    def _apply_1q_unchecked(self, q: int, m) -> None:
        global amplitude_writes
        self._axis(q)
        call("sk_apply_1q", self._h, q, _lib.mat8(_as_mat(m)))
        amplitude_writes += 1 << self.width

    def apply_controlled(self, controls, polarity, target: int, m) -> None:
        """Apply m to target where control bits match polarity (ket.py:146-164)."""
        global amplitude_writes
        controls, polarity = tuple(controls), tuple(polarity)
        qubits = controls + (target,)
        if len(set(qubits)) != len(qubits):
            raise ValueError(f"overlapping qubit indices {qubits}")
        m = _as_mat(m)
        _check_unitary(m)
        mask = val = 0
        for c, pol in zip(controls, polarity):
            self._axis(c)
            mask |= 1 << c
            if pol:
                val |= 1 << c
        self._axis(target)
        call("sk_apply_controlled", self._h, mask, val, target, _lib.mat8(m))
        amplitude_writes += 2 * (1 << (self.width - 1 - len(set(c for c, _ in zip(controls, polarity)))))

    def apply_controlled_bloch(self, control: int, polarity: int, target: int, m):
        """One-control gate fused with both operands' Bloch vectors
        (engine.py:389-394 runs apply_controlled then two bloch_vector passes).
        Returns (bloch of control, bloch of target) after the gate."""
        global amplitude_writes
        if control == target:
            raise ValueError(f"overlapping qubit indices {(control, target)}")
        m = _as_mat(m)
        _check_unitary(m)
        self._axis(control)
        self._axis(target)
        out = (C.c_double * 8)()
        call("sk_apply_controlled_bloch", self._h, control, int(polarity), target, _lib.mat8(m), out)
        amplitude_writes += 1 << (self.width - 1)
        return bloch_from_sums(out[0:4]), bloch_from_sums(out[4:8])

    def apply_controlled_bloch_sums(self, control: int, polarity: int, target: int, m):
        """As `apply_controlled_bloch` but returning the raw sums
        (Re, Im of sum conj(a0) a1, sum |a0|^2, sum |a1|^2) of control and target."""
        global amplitude_writes
        if control == target:
            raise ValueError(f"overlapping qubit indices {(control, target)}")
        m = _as_mat(m)
        _check_unitary(m)
        self._axis(control)
        self._axis(target)
        out = (C.c_double * 8)()
        call("sk_apply_controlled_bloch", self._h, control, int(polarity), target, _lib.mat8(m), out)
        amplitude_writes += 1 << (self.width - 1)
        return tuple(out[0:4]), tuple(out[4:8])

    def apply_pauli_layer(self, ops) -> None:
        """Simultaneous Paulis [(qubit, 'x'|'y'|'z'), ...] in one pass (ket.py:166-202)."""
        global amplitude_writes
        qubits = [q for q, _ in ops]
        if len(set(qubits)) != len(qubits):
            raise ValueError(f"duplicate qubit in pauli layer {qubits}")
        flip = sign = y_count = 0
        for q, p in ops:
            self._axis(q)
            if p == "x":
                flip |= 1 << q
            elif p == "y":
                flip |= 1 << q
                sign |= 1 << q
                y_count += 1
            elif p == "z":
                sign |= 1 << q
            else:
                raise ValueError(f"unknown pauli {p!r}")
        scale = 1j ** (y_count % 4)
        call("sk_apply_pauli_layer", self._h, flip, sign, scale.real, scale.imag)
        amplitude_writes += 1 << self.width

    def scale(self, z: complex) -> None:
        """amps *= z on the device (engine.py:706, tableau.py:279)."""
        z = complex(z)
        call("sk_scale", self._h, z.real, z.imag)

    def swap_qubits(self, a: int, b: int) -> None:
        """Exchange qubits a and b in place (tableau.py `_swap_bits`)."""
        self._axis(a)
        self._axis(b)
        call("sk_swap_qubits", self._h, a, b)

    def _bloch_sums(self, q: int):
        out = (C.c_double * 4)()
        call("sk_bloch_sums", self._h, q, out)
        return tuple(out)

    def bloch_vector(self, q: int) -> BlochVector:
        """(<X>, <Y>, <Z>) of qubit q from one pass (ket.py:204-210)."""
        self._axis(q)
        return bloch_from_sums(self._bloch_sums(q))

    def project_and_renormalize(self, q: int, outcome: int) -> float:
        """Project q onto outcome, rescale to unit norm, return the
        pre-projection probability (ket.py:212-226)."""
        global amplitude_writes
        if outcome not in (0, 1):
            raise ValueError(f"outcome must be 0 or 1, got {outcome}")
        self._axis(q)
        prob = C.c_double()
        call("sk_project", self._h, q, outcome, C.byref(prob))
        amplitude_writes += 1 << self.width
        return float(prob.value)

    def probability(self, q: int, outcome: int) -> float:
        self._axis(q)
        s = self._bloch_sums(q)
        return float(s[2] if outcome == 0 else s[3])

    def amplitude(self, index: int) -> complex:
        n = 1 << self.width
        if index < 0:
            index += n
        if not 0 <= index < n:
            raise IndexError(f"index {index} out of range for {n} amplitudes")
        out = (C.c_double * 2)()
        call("sk_amplitude", self._h, index, out)
        return complex(out[0], out[1])

    # ------------------------------------------------------------------
    # composition and factorisation
    # ------------------------------------------------------------------
    def kron_compose(self, other: "DenseKet") -> "DenseKet":
        """Tensor product; self keeps the low-order positions (ket.py:239-241)."""
        h = C.c_void_p()
        call("sk_kron", self._h, other._h, C.byref(h), needed=1 << (self.width + other.width))
        return self._new(h, self.width + other.width)

    def _compact(self, q: int, half: int, z: complex = 1.0) -> "DenseKet":
        h = C.c_void_p()
        z = complex(z)
        call("sk_compact", self._h, q, half, z.real, z.imag, C.byref(h), needed=1 << (self.width - 1))
        return self._new(h, self.width - 1)

    def try_decompose(self, q: int, tol: float):
        """Split q out as an exact (within tol) single-qubit factor (ket.py:243-267).

        One reduction pass gives the Bloch sums; the factor phi follows from
        them analytically (<dominant|a0>, <dominant|a1> are n0 / cross or
        conj(cross) / n1), and one compaction pass builds the remainder."""
        if self.width < 2:
            return None
        if tol < 0:
            raise ValueError("tolerance must be >= 0")
        self._axis(q)
        cr, ci, n0, n1 = self._bloch_sums(q)
        if epsilon_from_bloch(BlochVector(2 * cr, 2 * ci, n0 - n1)) > tol:
            return None
        cross = complex(cr, ci)
        if n0 >= 0.5:
            half, ndom, phi = 0, n0, np.array([n0, cross], dtype=complex)
        else:
            half, ndom, phi = 1, n1, np.array([cross.conjugate(), n1], dtype=complex)
        phi /= np.sqrt(np.sum(np.abs(phi) ** 2))
        rest = self._compact(q, half, 1.0 / math.sqrt(ndom))
        return DenseKet(1, phi, dtype=self.dtype, device=self.device), rest

    def remove_qubit(self, q: int) -> "DenseKet":
        """Drop qubit q, assumed exactly |0> (ket.py:269-275)."""
        self._axis(q)
        residual = self._bloch_sums(q)[3]
        if residual > 1e-9:
            raise ValueError(f"qubit {q} is not in |0> (residual {residual:.3e})")
        return self._compact(q, 0, 1.0)

    def round_qubit(self, q: int, u, scale: float) -> "DenseKet":
        """Fused SDRP step (engine.py:464-488): rest[k] = (u00 a0[k] + u01 a1[k]) * scale."""
        global amplitude_writes
        self._axis(q)
        u = _as_mat(u)
        h = C.c_void_p()
        u0 = _lib.darr((u[0, 0].real, u[0, 0].imag, u[0, 1].real, u[0, 1].imag))
        call("sk_round_compact", self._h, q, u0, float(scale), C.byref(h), needed=1 << (self.width - 1))
        amplitude_writes += 1 << self.width
        return self._new(h, self.width - 1)

    def split_measured(self, q: int, outcome: int, prob: float) -> "DenseKet":
        """Project q onto outcome and compact it away in one pass
        (engine.py:584-593: project_and_renormalize + remove_qubit)."""
        global amplitude_writes
        self._axis(q)
        amplitude_writes += 1 << self.width
        return self._compact(q, outcome, 1.0 / math.sqrt(prob))

    def fidelity(self, other: "DenseKet") -> float:
        """|<self|other>|^2 (ket.py:277-281)."""
        if self.width != other.width:
            raise ValueError(f"width mismatch: {self.width} vs {other.width}")
        if other.dtype != self.dtype:
            other = DenseKet(other.width, other.amps, dtype=self.dtype, device=self.device)
        out = (C.c_double * 2)()
        call("sk_vdot", self._h, other._h, out)
        return float(out[0] ** 2 + out[1] ** 2)

    def vdot(self, other: "DenseKet") -> complex:
        out = (C.c_double * 2)()
        call("sk_vdot", self._h, other._h, out)
        return complex(out[0], out[1])

    def sample_indices(self, uniforms) -> np.ndarray:
        """Basis indices for host-drawn uniforms exactly as numpy's
        Generator.choice(p=|a|^2/sum) maps them (cumsum, normalise,
        searchsorted side='right'); engine.py:613-615, 648-650."""
        u = np.ascontiguousarray(uniforms, dtype=np.float64).reshape(-1)
        out = np.empty(u.size, dtype=np.int64)
        call("sk_sample", self._h, u.ctypes.data_as(_lib.dptr), u.size,
             out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def __repr__(self) -> str:
        return f"DenseKet(width={self.width}, dtype={self.dtype}, device={self.device})"


def permute_qubits(ket: DenseKet, order) -> DenseKet:
    """Reorder qubits: new qubit k is old qubit order[k] (ket.py:284-292)."""
    order = list(order)
    if sorted(order) != list(range(ket.width)):
        raise ValueError(f"order must be a permutation of 0..{ket.width - 1}")
    h = C.c_void_p()
    arr = (C.c_int * len(order))(*order)
    call("sk_permute", ket._h, arr, C.byref(h), needed=1 << ket.width)
    return ket._new(h, ket.width)
