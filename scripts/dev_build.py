"""Development build: sk_fused.cu with -DSK_DEV_SWEEP_ONLY (c64 generic LEAN
sweeps only, ~1/5 of the compile time) linked with the regular objects into
libshardcu.so.  Leaves build/DEV_LIB so the next regular build rebuilds."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2304_14969_b200 import _build as B  # noqa: E402

objdir = B.ROOT / "build" / "obj"
dev = B.ROOT / "build" / "dev"
dev.mkdir(parents=True, exist_ok=True)
nvcc = B._nvcc()
extra = sys.argv[1:]
fused = dev / "sk_fused.o"
subprocess.run([nvcc, *B.ARCH, *B.FLAGS, "-DSK_DEV_SWEEP_ONLY", *extra, "-c", str(B.CSRC / "sk_fused.cu"),
                "-o", str(fused)], check=True)
objs = [fused if s.stem == "sk_fused" else objdir / (s.stem + ".o") for s in B.sources()]
B.DEV_MARKER.parent.mkdir(parents=True, exist_ok=True)
B.DEV_MARKER.write_text("dev")
subprocess.run([nvcc, *B.ARCH, "-shared", "-o", str(B.LIB), *map(str, objs)], check=True)
print(B.LIB)
