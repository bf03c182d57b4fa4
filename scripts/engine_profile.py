"""54q x 7 SDRP engine runs (p = 0.6, the 2^26 budget): wall time per run and
per min-SDRP search, with the default flags (tableau shards) and without.
Under `ncu --metrics gpu__time_duration.sum` the launch list gives the GPU
busy time of the same runs."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2304_14969_b200.circuit import build_random_circuit, derive_seed  # noqa: E402
from paper_2304_14969_b200.engine import EngineConfig, OptFlags  # noqa: E402
from paper_2304_14969_b200.sdrp import min_sdrp_search, run_hybrid  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = build_random_circuit(54, 7, derive_seed(0, 0))
for flags in (OptFlags(), OptFlags(stabilizer_hybrid=False)):
    cfg = EngineConfig(sdrp=0.6, mem_budget=1 << 26, rng_seed=1, optimizations=flags)
    run_hybrid(c, cfg).flush_all()
    t0 = time.perf_counter()
    for _ in range(reps):
        sim = run_hybrid(c, cfg)
        sim.flush_all()
    dt = (time.perf_counter() - t0) / reps
    print(f"stabilizer_hybrid={flags.stabilizer_hybrid}: {dt * 1e3:.2f} ms per run, stats {sim.stats}", flush=True)
t0 = time.perf_counter()
for i in range(4):
    min_sdrp_search(54, 7, derive_seed(0, i), 1 << 26)
print(f"min-SDRP search 54q x7 at 2^26 (default flags): {(time.perf_counter() - t0) / 4:.4f} s per circuit")
