"""SDRP drivers over the device engine (the reference's validate.py:114-300
callers of the hot path): run a circuit through the hybrid engine, the exact
overlap fidelity against the fused dense executor, and the minimum-SDRP
search that config 5 (54 qubits, 7-10 layers) is quoted on."""
from __future__ import annotations

import time
from dataclasses import dataclass

from .circuit import Circuit, build_random_circuit
from .engine import EngineConfig, HybridState
from .errors import MemoryBudgetError
from .executor import dense_reference
from .ket import DenseKet

DEFAULT_P_STEP = 0.025


def run_hybrid(c: Circuit, cfg: EngineConfig, initial: DenseKet | None = None, group=None,
               local_max_width: int | None = None) -> HybridState:
    """validate.py:114-121.  With `local_max_width` (inside an initialised
    torch.distributed group, every rank calling it) the largest shard is
    split over the ranks once wider than that (sk_engine_set_distributed)."""
    sim = HybridState(c.width, cfg, group=group, local_max_width=local_max_width)
    if initial is not None:
        sim.load_state(initial)
    sim.apply_circuit(c)
    return sim


def exact_fidelity(c: Circuit, cfg: EngineConfig) -> tuple[float, float]:
    """(exact overlap with the plain dense simulation, engine estimate); validate.py:124-128."""
    exact = dense_reference(c, dtype=cfg.dtype)
    sim = run_hybrid(c, cfg)
    return sim.full_ket().fidelity(exact), sim.estimated_fidelity()


@dataclass(frozen=True)
class MinSdrpResult:
    feasible: bool
    p_min: float | None
    f_model: float | None
    peak_amplitudes: int = 0


@dataclass
class SdrpRun:
    p: float
    ok: bool
    f_model: float | None
    peak_amplitudes: int
    rounds: int
    wall_s: float


def min_sdrp_search(width: int, depth: int, seed: int, mem_budget: int, p_step: float = DEFAULT_P_STEP,
                    dtype: str = "c128", trace: list | None = None, group=None,
                    local_max_width: int | None = None) -> MinSdrpResult:
    """Lower p from 1 in p_step decrements until the budget fails; report the
    last completing run (validate.py:280-300)."""
    if p_step <= 0:
        raise ValueError("p_step must be > 0")
    c = build_random_circuit(width, depth, seed)
    best = None
    steps = int(round(1.0 / p_step))
    for i in range(steps, -1, -1):
        p = round(i * p_step, 9)
        cfg = EngineConfig(sdrp=p, mem_budget=mem_budget, rng_seed=seed, dtype=dtype)
        t0 = time.perf_counter()
        try:
            sim = run_hybrid(c, cfg, group=group, local_max_width=local_max_width)
            sim.flush_all()
        except MemoryBudgetError as exc:
            if trace is not None:
                trace.append(SdrpRun(p, False, None, exc.needed, 0, time.perf_counter() - t0))
            return best if best is not None else MinSdrpResult(False, None, None)
        if trace is not None:
            trace.append(SdrpRun(p, True, sim.estimated_fidelity(), sim.peak_amplitudes, len(sim.eps_record),
                                 time.perf_counter() - t0))
        best = MinSdrpResult(True, p, sim.estimated_fidelity(), sim.peak_amplitudes)
        if p == 0.0:
            break
    return best


def _search_worker(args):
    width, depth, seed, budget, p_step, dtype, device = args
    from .ket import set_default_device
    set_default_device(device)
    t0 = time.perf_counter()
    r = min_sdrp_search(width, depth, seed, budget, p_step, dtype)
    return seed, r, time.perf_counter() - t0


def min_sdrp_ensemble(width: int, depth: int, n_circuits: int, base_seed: int, mem_budget: int,
                      workers: int = 1, p_step: float = DEFAULT_P_STEP, dtype: str = "c128",
                      devices: list[int] | None = None):
    """min_sdrp_search over circuits derive_seed(base_seed, i), i < n_circuits,
    spread over `workers` processes (the reference's process-pool sweep,
    validate.py:203-204,223-229).  The searches are host-bound on the small
    shards of 54-qubit SDRP, so several processes share one GPU well; with
    `devices` they are dealt round-robin over GPUs.  Returns
    [(seed, MinSdrpResult, wall_s)] in circuit order."""
    from .circuit import derive_seed
    devices = devices or [0]
    jobs = [(width, depth, derive_seed(base_seed, i), mem_budget, p_step, dtype, devices[i % len(devices)])
            for i in range(n_circuits)]
    if workers <= 1:
        return [_search_worker(j) for j in jobs]
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as pool:
        return list(pool.map(_search_worker, jobs))


@dataclass
class HeatmapCell:
    """Ensemble mean fidelity estimate at one (p, depth) grid point (validate.py:244-252)."""

    p: float
    depth: int
    mean_f_model: float | None  # None when every run exceeded the budget
    completed: int
    failed: int


def sdrp_depth_heatmap(width: int, depths, p_grid, n_circuits: int, base_seed: int, mem_budget: int,
                       dtype: str = "c128") -> list[HeatmapCell]:
    """Fixed-p runs over a (p, depth) grid; budget failures are recorded, not
    searched around (validate.py:255-276)."""
    from .circuit import derive_seed
    cells = []
    for depth in depths:
        circuits = [build_random_circuit(width, depth, derive_seed(base_seed, depth, i)) for i in range(n_circuits)]
        for p in p_grid:
            total, done, failed = 0.0, 0, 0
            for i, c in enumerate(circuits):
                cfg = EngineConfig(sdrp=p, mem_budget=mem_budget, rng_seed=derive_seed(base_seed, depth, i),
                                   dtype=dtype)
                try:
                    sim = run_hybrid(c, cfg)
                    sim.flush_all()
                    total += sim.estimated_fidelity()
                    done += 1
                except MemoryBudgetError:
                    failed += 1
            cells.append(HeatmapCell(p, depth, total / done if done else None, done, failed))
    return cells
