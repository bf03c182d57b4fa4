"""Reference min-SDRP search (validate.py:280-300) over the paper-scale
ensemble seeds (54 qubits, depths 7..10, circuits derive_seed(0, i)), run on
the REFERENCE package in this container (test infrastructure: it produces the
CPU side of profiles/r02_sdrp54_paper.jsonl).

    python oracle/ref_sdrp_ensemble.py <budget_bits> <n_circuits> <procs> > out.jsonl
"""
from __future__ import annotations

import json
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")


def one(args):
    depth, i, budget_bits = args
    from shardsim import validate as rv
    seed = rv.derive_seed(0, i)
    t0 = time.perf_counter()
    r = rv.min_sdrp_search(54, depth, seed, 1 << budget_bits)
    return {"depth": depth, "i": i, "seed": seed, "budget_bits": budget_bits, "feasible": r.feasible,
            "p_min": r.p_min, "f_model": r.f_model, "peak": r.peak_amplitudes,
            "wall_s": time.perf_counter() - t0, "impl": "reference (shardsim, NumPy, 1 core)"}


if __name__ == "__main__":
    bits, n, procs = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    jobs = [(d, i, bits) for d in (7, 8, 9, 10) for i in range(n)]
    with ProcessPoolExecutor(procs) as ex:
        for rec in ex.map(one, jobs):
            print(json.dumps(rec), flush=True)
