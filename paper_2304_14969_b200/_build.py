"""Build libshardcu.so in-tree with nvcc for sm_100a.

The shared library is the product's only compute path; there is no CPU
fallback.  `build()` is called by __graft_entry__.build() and lazily by
`_lib.load()` when the .so is missing or older than its sources.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libshardcu.so"
ROOT = PKG.parent
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}"]


def device_code_sha256(lib: Path = LIB) -> str | None:
    """sha256 of the .nv_fatbin section (the sm_100a device code) of the
    library.  nvcc embeds temporary file names in host objects, so two builds
    of the same sources differ as files; their device code does not."""
    import hashlib
    import struct

    try:
        b = lib.read_bytes()
    except OSError:
        return None
    if b[:4] != b"\x7fELF" or b[4] != 2:  # 64-bit ELF only
        return None
    shoff, = struct.unpack_from("<Q", b, 0x28)
    shentsize, shnum, shstrndx = struct.unpack_from("<HHH", b, 0x3A)
    sec = [struct.unpack_from("<IIQQQQ", b, shoff + i * shentsize) for i in range(shnum)]
    stroff = sec[shstrndx][4]
    for name, _t, _f, _a, off, size in sec:
        end = b.index(b"\0", stroff + name)
        if b[stroff + name:end] == b".nv_fatbin":
            return hashlib.sha256(b[off:off + size]).hexdigest()
    return None


def kernel_sass_sha256(pattern: str = "k_qft", lib: Path = LIB) -> str | None:
    """sha256 of the SASS of the library's kernels whose name contains
    `pattern` (cuobjdump, addresses stripped).  The key the committed ncu
    summary is matched on: rebuilding identical sources has produced
    different .nv_fatbin bytes but identical kernel code."""
    import hashlib
    import re
    import shutil

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists() or not lib.exists():
        return None
    try:
        out = subprocess.run([tool, "-sass", str(lib)], capture_output=True, text=True, timeout=120).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    h = hashlib.sha256()
    keep = False
    n = 0
    for line in out.splitlines():
        if "Function : " in line:
            keep = pattern in line
            n += keep
        if keep:
            line = re.sub(r"/\*[0-9a-fx]+\*/", "", line).strip()
            if line:
                h.update(line.encode() + b"\n")
    return h.hexdigest() if n else None


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _deps(src: Path, seen: set | None = None) -> set:
    """src plus every header it #includes (transitively) from csrc/ and include/."""
    import re
    seen = set() if seen is None else seen
    if src in seen or not src.exists():
        return seen
    seen.add(src)
    for inc in re.findall(r'#include\s+"([^"]+)"', src.read_text(errors="ignore")):
        _deps((src.parent / inc).resolve(), seen)
    return seen


# scripts/dev_build.py links a reduced development library (c64 generic
# sweeps only); its marker forces the next regular build
DEV_MARKER = ROOT / "build" / "DEV_LIB"


def is_stale() -> bool:
    if not LIB.exists() or DEV_MARKER.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources() + headers())


def _obj_stale(src: Path, obj: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _deps(src.resolve()))


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not is_stale():
        return LIB
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        if not force and not _obj_stale(src, obj):
            return obj  # incremental: only sources whose own include closure changed
        cmd = [nvcc, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=4) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    DEV_MARKER.unlink(missing_ok=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
