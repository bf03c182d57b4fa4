"""Host-side phase timing of a 54q x 7 SDRP engine run (p = 0.6, 2^26) with
and without tableau shards: construction, apply_circuit, flush_all."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2304_14969_b200.circuit import build_random_circuit, derive_seed  # noqa: E402
from paper_2304_14969_b200.engine import EngineConfig, HybridState, OptFlags  # noqa: E402

c = build_random_circuit(54, 7, derive_seed(0, 0))
for stab in (True, False, True, False):
    cfg = EngineConfig(sdrp=0.6, mem_budget=1 << 26, rng_seed=1, optimizations=OptFlags(stabilizer_hybrid=stab))
    tt = [0.0, 0.0, 0.0]
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim = HybridState(c.width, cfg)
        t1 = time.perf_counter()
        sim.apply_circuit(c)
        t2 = time.perf_counter()
        sim.flush_all()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        tt = [tt[0] + t1 - t0, tt[1] + t2 - t1, tt[2] + t3 - t2]
    print(f"stab={stab}: create {tt[0] / 5 * 1e3:.2f} ms, apply {tt[1] / 5 * 1e3:.2f} ms, flush {tt[2] / 5 * 1e3:.2f} ms",
          flush=True)
