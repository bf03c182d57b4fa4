"""Wall time of a 54-qubit min-SDRP ensemble with 1 and W worker processes
sharing one GPU.  usage: python scripts/sdrp_ensemble.py [circuits] [workers...]"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2304_14969_b200.sdrp import min_sdrp_ensemble  # noqa: E402

if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    for w in [int(x) for x in sys.argv[2:]] or [1, 8]:
        t0 = time.perf_counter()
        res = min_sdrp_ensemble(54, 7, n, 0, 1 << 30, workers=w, dtype="c64")
        dt = time.perf_counter() - t0
        fs = [r.f_model if r.feasible else 0.0 for _, r, _ in res]
        print(json.dumps({"config": "sdrp54_ensemble", "depth": 7, "circuits": n, "workers": w, "cpus": os.cpu_count(),
                          "wall_s": dt, "s_per_circuit": dt / n, "f_model_mean": sum(fs) / n,
                          "p_min": [r.p_min for _, r, _ in res]}), flush=True)
