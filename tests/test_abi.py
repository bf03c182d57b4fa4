"""The C-ABI library loads on a GPU-less host and exports every entry point
include/shardcu.h declares (no compute calls here).  CPU only."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from paper_2304_14969_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "shardcu.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sk_\w+)\s*\(", text, re.M)))


def test_header_declares_the_binding():
    assert set(declared()) == set(_lib.EXPORTS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in declared():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr), name


def test_no_device_is_reported_not_faked():
    # on the CPU host: zero devices, and creating a state fails loudly
    n = _lib.device_count()
    assert n >= 0
    if n == 0:
        import pytest
        from paper_2304_14969_b200 import DenseKet, DeviceError
        with pytest.raises(DeviceError):
            DenseKet(3)


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.SkOp) == 4 * 4 + 8 * 2 + 8 * 8
    assert ctypes.sizeof(_lib.SkSweep) == 4 * (1 + 16 + 1 + 8 * 5 + 9 + 1)


def test_device_code_hash_reads_the_fatbin(tmp_path):
    """bench.py matches the committed ncu summary by the sha256 of the
    library's .nv_fatbin section (identical device code across rebuilds)."""
    from paper_2304_14969_b200 import _build

    h = _build.device_code_sha256()
    assert h is not None and len(h) == 64 and int(h, 16) >= 0
    bogus = tmp_path / "not_elf.so"
    bogus.write_bytes(b"not an elf file")
    assert _build.device_code_sha256(bogus) is None


def test_kernel_sass_hash_is_stable_key():
    """The ncu summary is matched on the SASS of the k_qft kernels."""
    from paper_2304_14969_b200 import _build

    h = _build.kernel_sass_sha256("k_qft")
    if h is None:
        pytest.skip("cuobjdump not available")
    assert len(h) == 64 and h == _build.kernel_sass_sha256("k_qft")
    assert _build.kernel_sass_sha256("no_such_kernel_name") is None
