"""One 54q x 7 SDRP engine run (p = 0.6, 2^26) per flag setting, for an ncu
launch list: python scripts/engine_modes.py [stab|dense]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2304_14969_b200.circuit import build_random_circuit, derive_seed  # noqa: E402
from paper_2304_14969_b200.engine import EngineConfig, OptFlags  # noqa: E402
from paper_2304_14969_b200.sdrp import run_hybrid  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "stab"
c = build_random_circuit(54, 7, derive_seed(0, 0))
cfg = EngineConfig(sdrp=0.6, mem_budget=1 << 26, rng_seed=1,
                   optimizations=OptFlags(stabilizer_hybrid=(mode == "stab")))
run_hybrid(c, cfg).flush_all()
print("warm", flush=True)
sim = run_hybrid(c, cfg)
sim.flush_all()
print(mode, sim.stats)
