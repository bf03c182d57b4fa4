"""cProfile of one 54-qubit depth-7 SDRP run through the hybrid engine."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2304_14969_b200.circuit import build_random_circuit, derive_seed  # noqa: E402
from paper_2304_14969_b200.engine import EngineConfig  # noqa: E402
from paper_2304_14969_b200.sdrp import run_hybrid  # noqa: E402

c = build_random_circuit(54, 7, derive_seed(0, 0))
cfg = EngineConfig(sdrp=0.6, mem_budget=1 << 30, rng_seed=1, dtype="c64")
run_hybrid(c, cfg).flush_all()
t0 = time.perf_counter()
for _ in range(3):
    run_hybrid(c, cfg).flush_all()
print("per run", (time.perf_counter() - t0) / 3)
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    run_hybrid(c, cfg).flush_all()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

# per-entry-point wall time (each call returns after its stream work only if it synchronises)
import collections  # noqa: E402
from paper_2304_14969_b200 import _lib  # noqa: E402
acc = collections.defaultdict(lambda: [0, 0.0])
orig = _lib.call


def timed(name, *a, **kw):
    t = time.perf_counter()
    try:
        return orig(name, *a, **kw)
    finally:
        acc[name][0] += 1
        acc[name][1] += time.perf_counter() - t


_lib.call = timed
import paper_2304_14969_b200.ket as K  # noqa: E402
import paper_2304_14969_b200.engine as EN  # noqa: E402
K.call = timed  # ket.py binds `call` at import
for _ in range(3):
    run_hybrid(c, cfg).flush_all()
for k, (n, t) in sorted(acc.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} calls/run {n / 3:8.1f}  ms/run {t / 3 * 1e3:8.2f}  us/call {t / max(n, 1) * 1e6:8.1f}")
