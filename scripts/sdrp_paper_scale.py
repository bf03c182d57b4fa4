"""Paper-scale SDRP ensemble (BASELINE configs[4]):
min-SDRP search (validate.py:280-300) on 54-qubit random circuits, depths
7..10, circuits derive_seed(0, i), i < n, on the device engine.

Two legs per circuit, one JSON line each (flushed as it goes):
  * budget 2^22, c128: the same search the reference CPU runs
    (oracle/ref_sdrp_ensemble.py), for decision parity (p_min, F_model, peak);
  * the device budget (default 2^33 amplitudes, c64 = 64 GiB of shards plus
    merge transients): what one B200 reaches.

    python scripts/sdrp_paper_scale.py [n_circuits] [device_budget_bits] [minutes]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2304_14969_b200.circuit import derive_seed  # noqa: E402
from paper_2304_14969_b200.sdrp import min_sdrp_search  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
big = int(sys.argv[2]) if len(sys.argv) > 2 else 33
minutes = float(sys.argv[3]) if len(sys.argv) > 3 else 40.0
out = ROOT / "gpurun_out" / "sdrp54_paper.jsonl"
out.parent.mkdir(exist_ok=True)
deadline = time.time() + 60 * minutes
min_sdrp_search(54, 7, derive_seed(0, 999), 1 << 20)  # warm-up (context, pools)
with out.open("a") as fh:
    for i in range(n):
        for depth in (7, 8, 9, 10):
            if time.time() > deadline:
                sys.exit(0)
            seed = derive_seed(0, i)
            for bits, dtype in ((22, "c128"), (big, "c64")):
                t0 = time.perf_counter()
                r = min_sdrp_search(54, depth, seed, 1 << bits, dtype=dtype)
                rec = {"depth": depth, "i": i, "seed": seed, "budget_bits": bits, "dtype": dtype,
                       "feasible": r.feasible, "p_min": r.p_min, "f_model": r.f_model, "peak": r.peak_amplitudes,
                       "wall_s": time.perf_counter() - t0}
                fh.write(json.dumps(rec) + "\n")
                fh.flush()
