"""ctypes binding of libshardcu.so (the C ABI declared in include/shardcu.h).

There is deliberately no CPU fallback: if the library cannot be loaded, or no
CUDA device is visible when a state is created, the call raises.
"""
from __future__ import annotations

import ctypes as C
import threading

from . import _build
from .errors import DeviceError, DeviceMemoryError

SK_OK, SK_EINDEX, SK_EVALUE, SK_ENOMEM, SK_ECUDA, SK_EBUDGET = 0, 1, 2, 3, 4, 5
SK_C64, SK_C128 = 0, 1
SK_OP_MAT, SK_OP_DIAG, SK_OP_RAMP, SK_OP_QFT = 0, 1, 2, 3
SK_MAX_TILE_BITS, SK_MAX_REG_BITS, SK_MAX_STAGES = 16, 5, 8

DTYPES = {"c64": SK_C64, "complex64": SK_C64, "c128": SK_C128, "complex128": SK_C128}

_lib = None
_lock = threading.Lock()

p_state = C.c_void_p
p_prog = C.c_void_p
dptr = C.POINTER(C.c_double)


class SkOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("qubit", C.c_int32), ("nbits", C.c_int32), ("pad", C.c_int32),
                ("ctrl_mask", C.c_uint64), ("ctrl_val", C.c_uint64), ("m", C.c_double * 8)]


class SkSweep(C.Structure):
    _fields_ = [("ntile", C.c_int32), ("tile_bits", C.c_int32 * SK_MAX_TILE_BITS), ("nstages", C.c_int32),
                ("reg_bits", (C.c_int32 * SK_MAX_REG_BITS) * SK_MAX_STAGES),
                ("op_begin", C.c_int32 * (SK_MAX_STAGES + 1)), ("nreg", C.c_int32)]


class SkEngineConfig(C.Structure):
    _fields_ = [("sdrp", C.c_double), ("separability_tol", C.c_double), ("mem_budget", C.c_int64),
                ("dtype", C.c_int32), ("device", C.c_int32), ("control_elimination", C.c_int32),
                ("hx_commutation", C.c_int32), ("label_swap", C.c_int32), ("pauli_coalescing", C.c_int32),
                ("stabilizer_hybrid", C.c_int32)]


SK_GATE_1Q, SK_GATE_SWAP, SK_GATE_MEASURE = 0, 1, 2
ENGINE_STATS = ("label_swaps", "kernels", "eliminated_controls", "merges", "splits", "allocs", "amplitude_writes",
                "dense_total", "peak_amplitudes", "n_eps", "needed", "dist_shards", "exchanges")
UNIFORM_FN = C.CFUNCTYPE(C.c_double, C.c_void_p)
BIT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)
SENDRECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_int64)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64)
p_engine = C.c_void_p
i32p = C.POINTER(C.c_int32)

# name -> argtypes (restype is always c_int unless listed in _RESTYPES)
_SIGS = {
    "sk_last_error": [],
    "sk_version": [],
    "sk_device_count": [],
    "sk_set_stream": [C.c_int, C.c_uint64],
    "sk_get_stream": [C.c_int, C.POINTER(C.c_uint64)],
    "sk_synchronize": [C.c_int],
    "sk_mem_info": [C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
    "sk_create": [C.c_int, C.c_int, C.c_int, C.POINTER(p_state)],
    "sk_create_from": [C.c_int, C.c_int, C.c_int, dptr, C.POINTER(p_state)],
    "sk_copy": [p_state, C.POINTER(p_state)],
    "sk_destroy": [p_state],
    "sk_wrap": [C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(p_state)],
    "sk_rebind": [p_state, C.c_uint64],
    "sk_width": [p_state, C.POINTER(C.c_int)],
    "sk_dtype": [p_state, C.POINTER(C.c_int)],
    "sk_device_ptr": [p_state, C.POINTER(C.c_uint64)],
    "sk_upload": [p_state, dptr, C.c_int64],
    "sk_download": [p_state, dptr, C.c_int64],
    "sk_upload_native": [p_state, C.c_void_p, C.c_int64],
    "sk_download_native": [p_state, C.c_void_p, C.c_int64],
    "sk_download_native_async": [p_state, C.c_void_p, C.c_int64],
    "sk_copy_from_device": [p_state, C.c_uint64, C.c_int64],
    "sk_copy_to_device": [p_state, C.c_uint64, C.c_int64],
    "sk_apply_1q": [p_state, C.c_int, dptr],
    "sk_apply_controlled": [p_state, C.c_uint64, C.c_uint64, C.c_int, dptr],
    "sk_apply_controlled_bloch": [p_state, C.c_int, C.c_int, C.c_int, dptr, dptr],
    "sk_apply_pauli_layer": [p_state, C.c_uint64, C.c_uint64, C.c_double, C.c_double],
    "sk_scale": [p_state, C.c_double, C.c_double],
    "sk_swap_qubits": [p_state, C.c_int, C.c_int],
    "sk_bloch_sums": [p_state, C.c_int, dptr],
    "sk_norm2": [p_state, dptr],
    "sk_vdot": [p_state, p_state, dptr],
    "sk_amplitude": [p_state, C.c_int64, dptr],
    "sk_project": [p_state, C.c_int, C.c_int, dptr],
    "sk_compact": [p_state, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(p_state)],
    "sk_round_compact": [p_state, C.c_int, dptr, C.c_double, C.POINTER(p_state)],
    "sk_kron": [p_state, p_state, C.POINTER(p_state)],
    "sk_permute": [p_state, C.POINTER(C.c_int), C.POINTER(p_state)],
    "sk_sample": [p_state, dptr, C.c_int64, C.POINTER(C.c_int64)],
    "sk_program_reg_bits": [C.c_int, C.POINTER(C.c_int)],
    "sk_program_create": [C.c_int, C.c_int, C.c_int, C.POINTER(SkSweep), C.c_int, C.POINTER(SkOp), C.c_int,
                          C.POINTER(p_prog)],
    "sk_program_destroy": [p_prog],
    "sk_program_lower": [C.c_int, C.c_int, C.POINTER(SkSweep), C.c_int, C.POINTER(SkOp), C.c_int,
                         C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "sk_program_run": [p_state, p_prog, C.c_int, C.c_int],
    "sk_program_nsweeps": [p_prog, C.POINTER(C.c_int)],
    "sk_program_set_phase_index": [p_prog, C.c_int, C.c_uint64],
    "sk_program_run_tiles": [p_state, p_prog, C.c_int, C.c_int64, C.c_int64],
    "sk_program_sweep_tiles": [p_prog, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64)],
    "sk_engine_create": [C.c_int, C.POINTER(SkEngineConfig), C.POINTER(p_engine)],
    "sk_engine_destroy": [p_engine],
    "sk_engine_set_rng": [p_engine, UNIFORM_FN, C.c_void_p],
    "sk_engine_set_rng_bits": [p_engine, BIT_FN, C.c_void_p],
    "sk_engine_set_distributed": [p_engine, C.c_int, C.c_int, C.c_int, ALLREDUCE_FN, SENDRECV_FN, ALLGATHER_FN,
                                  C.c_void_p],
    "sk_engine_apply": [p_engine, C.c_int, i32p, i32p, i32p, i32p, i32p, dptr, C.POINTER(C.c_int)],
    "sk_engine_measure": [p_engine, C.c_int, C.POINTER(C.c_int)],
    "sk_engine_flush_all": [p_engine],
    "sk_engine_flush_qubit": [p_engine, C.c_int],
    "sk_engine_sdrp_round": [p_engine, C.c_int, C.c_double, dptr],
    "sk_engine_stats": [p_engine, C.POINTER(C.c_int64)],
    "sk_engine_eps": [p_engine, dptr, C.c_int64],
    "sk_engine_shards": [p_engine, C.c_int, C.POINTER(p_state), C.POINTER(C.c_int), C.POINTER(C.c_int),
                         C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "sk_engine_load_state": [p_engine, p_state],
    "sk_engine_measure_all": [p_engine, C.POINTER(C.c_uint8)],
    "sk_engine_sample": [p_engine, C.c_int64, C.POINTER(C.c_uint8)],
}
_RESTYPES = {"sk_last_error": C.c_char_p}

EXPORTS = tuple(_SIGS)


def load():
    """Load (building first if stale) and bind libshardcu.so."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if _build.is_stale():
            try:
                _build.build()
            except Exception as exc:  # no nvcc on this host: only a prebuilt .so can work
                if not path.exists():
                    raise ImportError(f"libshardcu.so missing and could not be built: {exc}") from exc
        lib = C.CDLL(str(path))
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().sk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, needed: int | None = None) -> None:
    """Map an SK_* status to the reference's exception types."""
    if rc == SK_OK:
        return
    msg = last_error()
    if rc == SK_EINDEX:
        raise IndexError(msg)
    if rc == SK_EVALUE:
        raise ValueError(msg)
    if rc == SK_ENOMEM:
        raise DeviceMemoryError(f"{msg} (needed {needed} amplitudes)" if needed is not None else msg)
    raise DeviceError(msg)


def call(name: str, *args, needed: int | None = None) -> None:
    check(getattr(load(), name)(*args), needed=needed)


def device_count() -> int:
    return int(load().sk_device_count())


def require_device() -> None:
    if device_count() < 1:
        raise DeviceError("libshardcu: no CUDA device visible (this engine has no CPU fallback)")


def darr(values) -> "C.Array":
    vals = [float(v) for v in values]
    return (C.c_double * len(vals))(*vals)


def mat8(m) -> "C.Array":
    """2x2 complex matrix -> double[8] (re/im of m00, m01, m10, m11)."""
    return darr((m[0][0].real, m[0][0].imag, m[0][1].real, m[0][1].imag,
                 m[1][0].real, m[1][0].imag, m[1][1].real, m[1][1].imag))
