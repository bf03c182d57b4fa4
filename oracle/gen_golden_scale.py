"""Generate tests/golden/scale_*.npz at the BASELINE configs' real sizes by
running the REFERENCE package itself (test infrastructure only).

Run here (the only place /root/reference exists), one part per process:
    python oracle/gen_golden_scale.py qft27      # ~3 min, ~10 GiB RSS
    python oracle/gen_golden_scale.py rand20
    python oracle/gen_golden_scale.py rand24     # ~3 min
    python oracle/gen_golden_scale.py sdrp54     # reference min_sdrp_search, 4 circuits x 2 budgets

The full outputs are far too large to commit, so each golden keeps
size-independent witnesses of the reference's output vector y:
  * `idx` / `amp`: y at 4096 seeded random indices (plus index 0 and N-1);
  * `chunk`: the sums of y over 256 equal contiguous chunks (a linear
    checksum of every amplitude);
  * `norm2`: sum |y|^2.
Inputs are regenerated bit-identically on the GPU box from the stored seed
with numpy's PCG64 (`random_state`, the reference's conftest.py:8-10
construction), so the test feeds the device exactly the reference's input.

Reference calls: validate.dense_reference (validate.py:83-111) with its CPU
cap DENSE_BUDGET (validate.py:22) lifted to the workload size for QFT-27 —
the loop itself is unmodified; validate.min_sdrp_search (validate.py:280-300)
and run_hybrid (:114-121) for the 54-qubit SDRP decisions.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
N_SAMPLES = 4096
N_CHUNKS = 256


def random_state(width: int, seed: int) -> np.ndarray:
    """conftest.py:8-10: normal + 1j*normal, normalised (PCG64 default_rng)."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << width) + 1j * rng.normal(size=1 << width)
    v /= np.linalg.norm(v)
    return v


def sample_indices(width: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed + 7919)
    idx = rng.integers(0, 1 << width, size=N_SAMPLES, dtype=np.int64)
    return np.unique(np.concatenate([idx, [0, (1 << width) - 1]]))


def witnesses(y: np.ndarray, width: int, seed: int, prefix: str) -> dict:
    idx = sample_indices(width, seed)
    return {f"{prefix}/idx": idx, f"{prefix}/amp": y[idx],
            f"{prefix}/chunk": y.reshape(N_CHUNKS, -1).sum(axis=1),
            f"{prefix}/norm2": float(np.vdot(y, y).real)}


def gen_qft27() -> dict:
    from shardsim import circuit as rc
    from shardsim import ket as rk
    from shardsim import validate as rv

    n, seed = 27, 2027
    x = random_state(n, seed)
    rv.DENSE_BUDGET = 1 << n  # lift the CPU cap only; the loop is the reference's own
    t0 = time.time()
    y = rv.dense_reference(rc.build_qft(n), initial=rk.DenseKet(n, x)).amps
    dt = time.time() - t0
    d = witnesses(y, n, seed, "qft27")
    d["qft27/spec"] = np.array([n, seed], dtype=np.int64)
    d["qft27/ref_seconds"] = dt
    # independent cross-check of the golden itself: numpy's FFT (positive exponent = ifft * sqrt(N))
    f = np.fft.ifft(x) * np.sqrt(x.size)
    d["qft27/fft_maxdiff"] = float(np.max(np.abs(f - y)))
    print(f"qft27: reference {dt:.1f} s, |ref - fft|max = {d['qft27/fft_maxdiff']:.3e}")
    return d


def gen_rand(width: int) -> dict:
    from shardsim import circuit as rc
    from shardsim import validate as rv

    depth, seed = 20, rv.derive_seed(0, width)
    t0 = time.time()
    y = rv.dense_reference(rc.build_random_circuit(width, depth, seed)).amps
    dt = time.time() - t0
    key = f"rand{width}"
    d = witnesses(y, width, seed & 0x7FFFFFFF, key)
    d[f"{key}/spec"] = np.array([width, depth, seed], dtype=np.uint64)
    d[f"{key}/ref_seconds"] = dt
    print(f"{key}: reference {dt:.1f} s")
    return d


def gen_sdrp54() -> dict:
    """Reference min-SDRP search (validate.py:280-300) on 54q x 7 circuits
    0..3 at 2^20 and 2^22 amplitude budgets, then the p_min run's eps record
    and peak (run_hybrid + flush_all as the search does)."""
    from shardsim import circuit as rc
    from shardsim import engine as reng
    from shardsim import validate as rv

    d = {}
    for budget_bits in (20, 22):
        for i in range(4):
            seed = rv.derive_seed(0, i)
            t0 = time.time()
            r = rv.min_sdrp_search(54, 7, seed, 1 << budget_bits)
            dt = time.time() - t0
            key = f"sdrp54/{i}_{budget_bits}"
            d[f"{key}/spec"] = np.array([54, 7, seed, 1 << budget_bits], dtype=np.uint64)
            d[f"{key}/res"] = np.array([r.feasible, -1 if r.p_min is None else r.p_min,
                                        -1 if r.f_model is None else r.f_model,
                                        -1 if r.peak_amplitudes is None else r.peak_amplitudes], dtype=float)
            d[f"{key}/ref_seconds"] = dt
            if r.feasible:
                sim = rv.run_hybrid(rc.build_random_circuit(54, 7, seed),
                                    reng.EngineConfig(sdrp=r.p_min, mem_budget=1 << budget_bits, rng_seed=seed))
                sim.flush_all()
                d[f"{key}/eps"] = np.array(sim.eps_record)
                d[f"{key}/stats"] = np.array([sim.stats[k] for k in ("label_swaps", "kernels", "eliminated_controls",
                                                                     "merges", "splits")])
            print(f"{key}: p_min={r.p_min} F={r.f_model} peak={r.peak_amplitudes} ({dt:.1f} s)")
    return d


if __name__ == "__main__":
    part = sys.argv[1]
    OUT.mkdir(parents=True, exist_ok=True)
    if part == "qft27":
        d = gen_qft27()
    elif part.startswith("rand"):
        d = gen_rand(int(part[4:]))
    elif part == "sdrp54":
        d = gen_sdrp54()
    else:
        raise SystemExit(f"unknown part {part}")
    path = OUT / f"scale_{part}.npz"
    np.savez_compressed(path, **d)
    print(path, path.stat().st_size)
