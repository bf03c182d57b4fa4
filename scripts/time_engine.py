"""Wall time per 54q x 7 SDRP run (p=0.6, c64) through the hybrid engine."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2304_14969_b200.circuit import build_random_circuit, derive_seed  # noqa: E402
from paper_2304_14969_b200.engine import EngineConfig  # noqa: E402
from paper_2304_14969_b200.sdrp import run_hybrid  # noqa: E402

c = build_random_circuit(54, 7, derive_seed(0, 0))
for p in (0.6, 0.55):
    cfg = EngineConfig(sdrp=p, mem_budget=1 << 33, rng_seed=1, dtype="c64")
    sim = run_hybrid(c, cfg)
    sim.flush_all()
    for trial in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            sim = run_hybrid(c, cfg)
            sim.flush_all()
        torch.cuda.synchronize()
        print(f"p={p} trial {trial}: {(time.perf_counter() - t0) / 5 * 1e3:.1f} ms per run, peak {sim.peak_amplitudes}",
              flush=True)
