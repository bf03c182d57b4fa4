"""Command-line reporting surface for the device engine.

Mirrors the reference's `shardsim` CLI (cli.py:76-236, 281-344) for the
subcommands on the hot path, with the same arguments, CSV schemas, environment
stamp and exit codes (0 ok, 2 usage, 4 memory budget exceeded, 5 internal
error or failed verification).  Each CSV gains GPU columns: device, dtype,
fused sweeps, HBM GB/s and the fraction of the measured HBM peak.

    python -m paper_2304_14969_b200.cli qft-bench --n-min 20 --n-max 27 --engine fused
    python -m paper_2304_14969_b200.cli min-sdrp --width 54 --depths 7:10 --circuits 10 --i-have-80gb
    python -m paper_2304_14969_b200.cli validate --grid 6x6,12x6 --circuits 20

`qft-bench --engine hybrid` times the reference's own path (HybridState on
|0..0> or GHZ input, cli.py:87-98); `--engine fused` times the fused dense
executor on a resident state.  Verification uses the QFT's closed forms on
sampled amplitudes (|0> -> uniform; GHZ -> (1 + e^{-2 pi i j/N}) / sqrt(2N)):
for the fused engine at every width (relative tolerance), for the hybrid
engine with the reference's rule (<= 2^22 amplitudes, 1e-9 absolute).  Like
the reference, the hybrid engine on GHZ input fails that rule from 18 qubits
on: its exact-split test (eps <= 1e-10, engine.py:455-460) splits nearly
separable qubits, an O(sqrt(eps)) amplitude error — ours reproduces the
reference's 3.310e-08 (n=18) and 3.511e-08 (n=19) with the same splits.  The `run` subcommand (circuit text files) is out
of scope with the text format.
"""
from __future__ import annotations

import argparse
import json
import math
import statistics
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import RNG_ALGORITHM, __version__ as VERSION

DEFAULT_BUDGET = 1 << 26  # the reference's DENSE_BUDGET (validate.py:22)
ORACLE_BUDGET = 1 << 22  # cli.py:39: above this the hybrid run is not verified
SWEEP_CSV_HEADER = "width,depth,seed,p,f_model,f_exact,wall_ms,peak_amplitudes"  # validate.py:166


@dataclass
class BenchReport:
    """Rows plus the environment stamp they were collected under (cli.py:42-61)."""

    experiment: str
    axes: dict
    header: str
    rows: list[str] = field(default_factory=list)
    notes: list[str] = field(default_factory=list)

    def stamp(self, seed: int, threads: int, device: str, dtype: str) -> list[str]:
        return [f"# engine=paper_2304_14969_b200 {VERSION}, rng={RNG_ALGORITHM}, threads={threads}, seed={seed}, "
                f"device={device}, dtype={dtype}",
                f"# experiment={self.experiment} " + " ".join(f"{k}={v}" for k, v in self.axes.items())]

    def write_csv(self, path: str, seed: int, threads: int, device: str, dtype: str) -> None:
        lines = self.stamp(seed, threads, device, dtype) + [self.header] + self.rows
        Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")


def _device_name() -> str:
    try:
        import torch
        return torch.cuda.get_device_name(0).replace(",", " ")
    except Exception:  # noqa: BLE001
        return "unknown"


def _hbm_peak() -> float:
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6553.9


def _sync(device: int = 0) -> None:
    from . import _lib
    _lib.call("sk_synchronize", device)


def _qft_expected(n: int, init: str, idx: np.ndarray) -> np.ndarray:
    N = float(1 << n)
    if init == "zero":
        return np.full(idx.size, 1.0 / math.sqrt(N), dtype=complex)
    return (1.0 + np.exp(-2j * np.pi * idx.astype(np.float64) / N)) / math.sqrt(2.0 * N)


def _verify(get_amp, n: int, init: str, dtype: str, samples: int = 512) -> float:
    rng = np.random.default_rng(n)
    idx = np.unique(np.concatenate([[0, (1 << n) - 1], rng.integers(0, 1 << n, samples)]))
    got = np.array([get_amp(int(i)) for i in idx])
    return float(np.max(np.abs(got - _qft_expected(n, init, idx))))


# ---------------------------------------------------------------------------
# qft-bench (cli.py:76-124)
# ---------------------------------------------------------------------------
def cmd_qft_bench(args) -> int:
    from .circuit import build_ghz, build_qft
    from .engine import EngineConfig, HybridState, OptFlags
    from .executor import compile_circuit
    from .ket import DenseKet, permute_qubits

    report = BenchReport("qft-bench", {"n_min": args.n_min, "n_max": args.n_max, "init": args.init,
                                       "repeats": args.repeats, "engine": args.engine},
                         "n,init,wall_ms,peak_amplitudes,verified,engine,sweeps,hbm_gbs,hbm_frac")
    rel_tol = 1e-9 if args.dtype == "c128" else 3e-5  # per amplitude, relative to |y_j| ~ 2^(-n/2)
    peak = _hbm_peak()
    for n in range(args.n_min, args.n_max + 1):
        times, sweeps, gbs, frac = [], "", "", ""
        if args.engine == "hybrid":
            sim = None
            for rep in range(args.repeats + 1):  # first run is a discarded warm-up
                sim = HybridState(n, EngineConfig(mem_budget=args.mem_budget, rng_seed=args.seed, dtype=args.dtype,
                                                  optimizations=OptFlags(stabilizer_hybrid=False)))
                if args.init == "ghz":
                    sim.apply_circuit(build_ghz(n))
                    sim.flush_all()
                _sync()
                t0 = time.monotonic()
                sim.apply_circuit(build_qft(n))
                sim.flush_all()
                _sync()
                if rep > 0:
                    times.append(time.monotonic() - t0)
            peak_amps = sim.peak_amplitudes
            # the reference's rule (cli.py:100-109): verify up to 2^22 amplitudes at 1e-9 absolute
            ket = sim.full_ket() if (1 << n) <= min(ORACLE_BUDGET, args.mem_budget) else None
            err = _verify(ket.amplitude, n, args.init, args.dtype) if ket is not None else None
        else:
            if (1 << n) > args.mem_budget:
                from .errors import MemoryBudgetError
                raise MemoryBudgetError(1 << n, args.mem_budget)
            prog = compile_circuit(build_qft(n), dtype=args.dtype)
            x = None
            if args.init == "ghz":
                x = np.zeros(1 << n, dtype=complex)
                x[0] = x[-1] = 2 ** -0.5
            for rep in range(args.repeats + 1):
                st = DenseKet(n, x, dtype=args.dtype)
                _sync()
                t0 = time.monotonic()
                prog.run(st)
                _sync()
                if rep > 0:
                    times.append(time.monotonic() - t0)
            peak_amps = 1 << n
            out = permute_qubits(st, prog.plan.order)
            err = _verify(out.amplitude, n, args.init, args.dtype)
            esz = 8 if args.dtype == "c64" else 16
            moved = prog.n_sweeps * 2 * esz * (1 << n)
            sweeps = str(prog.n_sweeps)
            g = moved / statistics.median(times) / 1e9
            gbs, frac = f"{g:.1f}", f"{g / peak:.3f}"
        wall_ms = statistics.median(times) * 1000
        limit = 1e-9 if args.engine == "hybrid" else rel_tol * 2.0 ** (-n / 2)
        verified = "" if err is None else ("1" if err < limit else "0")
        if verified == "0":
            report.notes.append(f"n={n}: closed-form mismatch {err:.3e}")
        report.rows.append(f"{n},{args.init},{wall_ms:.3f},{peak_amps},{verified},{args.engine},{sweeps},{gbs},{frac}")
        print(f"n={n:3d} init={args.init} engine={args.engine} wall_ms={wall_ms:.3f} peak={peak_amps} "
              f"verified={verified or '-'}" + (f" sweeps={sweeps} hbm={gbs} GB/s ({frac})" if sweeps else ""))
    report.write_csv(args.out, args.seed, 1, _device_name(), args.dtype)
    for note in report.notes:
        print(f"error: verification: {note}", file=sys.stderr)
    return 5 if report.notes else 0


# ---------------------------------------------------------------------------
# min-sdrp (cli.py:184-236)
# ---------------------------------------------------------------------------
def _parse_span(text: str) -> list[int]:
    if ":" in text:
        lo, _, hi = text.partition(":")
        return list(range(int(lo), int(hi) + 1))
    return [int(p) for p in text.split(",")]


def cmd_min_sdrp(args) -> int:
    from .sdrp import min_sdrp_ensemble

    if args.width >= 54 and not args.i_have_80gb:
        print("error: usage: width >= 54 needs tens of GB of amplitude storage; pass --i-have-80gb to acknowledge",
              file=sys.stderr)
        return 2
    if args.heatmap:  # cli.py:192-210
        from .sdrp import sdrp_depth_heatmap
        p_grid = [round(0.1 * k, 6) for k in range(1, 11)]
        cells = sdrp_depth_heatmap(args.width, _parse_span(args.depths), p_grid, args.circuits, args.seed,
                                   args.mem_budget, dtype=args.dtype)
        report = BenchReport("min-sdrp-heatmap", {"width": args.width, "circuits": args.circuits},
                             "p,depth,mean_f_model,completed,failed")
        for c in cells:
            mean = "" if c.mean_f_model is None else f"{c.mean_f_model:.12g}"
            report.rows.append(f"{c.p:.12g},{c.depth},{mean},{c.completed},{c.failed}")
        report.write_csv(args.out, args.seed, 1, _device_name(), args.dtype)
        return 0
    report = BenchReport("min-sdrp", {"width": args.width, "circuits": args.circuits, "mem_budget": args.mem_budget},
                         "width,depth,seed,p_min,f_model,peak_amplitudes,wall_ms")
    for depth in _parse_span(args.depths):
        values = []
        results = min_sdrp_ensemble(args.width, depth, args.circuits, args.seed, args.mem_budget,
                                    workers=args.threads, dtype=args.dtype)
        for seed, res, wall_s in results:
            wall_ms = wall_s * 1000
            if not res.feasible:
                report.rows.append(f"{args.width},{depth},{seed},,,,{wall_ms:.1f}")
                continue
            report.rows.append(f"{args.width},{depth},{seed},{res.p_min:.12g},{res.f_model:.12g},"
                               f"{res.peak_amplitudes},{wall_ms:.1f}")
            values.append(res.f_model)
        mean = sum(values) / len(values) if values else None
        shown = "infeasible" if mean is None else f"{mean:.4g}"
        print(f"depth={depth:3d} circuits={len(values)} mean_f_model={shown}")
    report.write_csv(args.out, args.seed, args.threads, _device_name(), args.dtype)
    return 0


# ---------------------------------------------------------------------------
# validate (cli.py:139-165; validate.py:166-212 without the process pool)
# ---------------------------------------------------------------------------
def _parse_grid(text: str) -> list[tuple[int, int]]:
    cells = []
    for part in text.split(","):
        w, _, d = part.strip().partition("x")
        cells.append((int(w), int(d)))
    return cells


def cmd_validate(args) -> int:
    from .circuit import build_random_circuit, derive_seed
    from .engine import EngineConfig
    from .errors import MemoryBudgetError
    from .executor import dense_reference
    from .sdrp import run_hybrid

    grid = [round(i * 0.025, 6) for i in range(41)] if args.p_grid is None else [float(p) for p in args.p_grid.split(",")]
    report = BenchReport("validate", {"grid": args.grid, "circuits": args.circuits}, SWEEP_CSV_HEADER)
    all_pairs, table = [], []
    for width, depth in _parse_grid(args.grid):
        base = derive_seed(args.seed, width, depth)
        pairs = []
        for i in range(args.circuits):
            seed = derive_seed(base, i)
            c = build_random_circuit(width, depth, seed)
            exact = dense_reference(c, dtype=args.dtype)
            for p in grid:
                t0 = time.monotonic()
                try:
                    sim = run_hybrid(c, EngineConfig(sdrp=p, mem_budget=args.mem_budget, rng_seed=seed,
                                                     dtype=args.dtype))
                    sim.flush_all()
                    fm, fe = sim.estimated_fidelity(), sim.full_ket().fidelity(exact)
                    wall = int((time.monotonic() - t0) * 1000)
                    report.rows.append(f"{width},{depth},{seed},{p:.12g},{fm:.12g},{fe:.12g},{wall},"
                                       f"{sim.peak_amplitudes}")
                    pairs.append((fm, fe))
                except MemoryBudgetError as exc:
                    wall = int((time.monotonic() - t0) * 1000)
                    report.rows.append(f"{width},{depth},{seed},{p:.12g},,,{wall},{exc.needed}")
        r = _rmse(pairs)
        all_pairs.extend(pairs)
        table.append((width, depth, r))
        print(f"{width:3d} x {depth:<3d} circuits={args.circuits} rmse={r:.4f}")
    overall = _rmse(all_pairs)
    print(f"Overall rmse={overall:.4f}")
    report.write_csv(args.out, args.seed, args.threads, _device_name(), args.dtype)
    summary = BenchReport("validate-rmse", {"grid": args.grid}, "width,depth,circuits,rmse")
    summary.rows = [f"{w},{d},{args.circuits},{r:.6f}" for w, d, r in table]
    summary.rows.append(f"overall,,{args.circuits * len(table)},{overall:.6f}")
    summary.write_csv(_sibling(args.out, "_rmse"), args.seed, args.threads, _device_name(), args.dtype)
    return 0


def _rmse(pairs) -> float:
    """validate.py:131-139: an empty cell is an error (the CLI exits 5), not NaN."""
    pairs = list(pairs)
    if not pairs:
        raise ValueError("rmse needs at least one (estimate, exact) pair")
    return math.sqrt(sum((a - b) ** 2 for a, b in pairs) / len(pairs))


def _sibling(path: str, suffix: str) -> str:
    """cli.py:168-170."""
    stem, dot, ext = path.rpartition(".")
    return f"{stem}{suffix}.{ext}" if dot else f"{path}{suffix}"


# ---------------------------------------------------------------------------
# parser and entry point (cli.py:281-344)
# ---------------------------------------------------------------------------
def _add_common(p, out_default: str, dtype_default: str) -> None:
    """The reference's common flags (cli.py:281-287) plus --dtype."""
    p.add_argument("--seed", type=int, default=0, help="base 64-bit seed")
    p.add_argument("--threads", type=int, default=1, help="worker processes sharing the GPU (validate.py:223-229)")
    p.add_argument("--mem-budget", type=int, default=DEFAULT_BUDGET, help="max dense amplitudes per simulator")
    p.add_argument("--out", default=out_default, help="output CSV path")
    p.add_argument("--format", choices=("csv", "csv+svg"), default="csv",
                   help="csv+svg is accepted; the SVG plots (svgplot.py) are out of scope, only the CSV is written")
    p.add_argument("--dtype", choices=("c64", "c128"), default=dtype_default, help="amplitude precision")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2304_14969_b200", description="B200 ket engine (shardsim drop-in)")
    sub = ap.add_subparsers(dest="command", required=True)

    p = sub.add_parser("qft-bench", help="Fourier-circuit timing benchmark")
    p.add_argument("--n-min", type=int, default=4)
    p.add_argument("--n-max", type=int, default=20)
    p.add_argument("--init", choices=("zero", "ghz"), default="zero")
    p.add_argument("--repeats", type=int, default=5)
    p.add_argument("--engine", choices=("hybrid", "fused"), default="hybrid")
    _add_common(p, "qft_bench.csv", "c128")
    p.set_defaults(func=cmd_qft_bench)

    p = sub.add_parser("validate", help="fidelity-model calibration sweep")
    p.add_argument("--grid", default="6x6,12x6,12x12,15x15", help="comma-separated width x depth cells")
    p.add_argument("--circuits", type=int, default=100)
    p.add_argument("--p-grid", default=None, help="comma-separated rounding parameters (default 0..1 by 0.025)")
    _add_common(p, "validate.csv", "c128")
    p.set_defaults(func=cmd_validate)

    p = sub.add_parser("min-sdrp", help="minimum rounding parameter search")
    p.add_argument("--width", type=int, default=16)
    p.add_argument("--depths", default="1:10", help="lo:hi or comma list")
    p.add_argument("--circuits", type=int, default=100)
    p.add_argument("--i-have-80gb", action="store_true", help="acknowledge the memory cost of width >= 54")
    p.add_argument("--heatmap", action="store_true", help="fixed p x depth cross-section instead of the search")
    _add_common(p, "min_sdrp.csv", "c128")
    p.set_defaults(func=cmd_min_sdrp)
    return ap


def main(argv=None) -> int:
    from .errors import InvariantError, MemoryBudgetError
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.func(args)
    except MemoryBudgetError as exc:
        print(f"error: budget: {exc}", file=sys.stderr)
        return 4
    except (InvariantError, Exception) as exc:  # noqa: BLE001
        print(f"error: internal: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 5


if __name__ == "__main__":
    sys.exit(main())
