"""Measure every BASELINE.json config on one B200 (device-timed, CUDA events
on the library stream) and print one JSON line per measurement.

  python scripts/bench_configs.py [qft20] [qft27] [rand30] [qft34] [sdrp54] [hybrid]

qft20/qft27: fused executor, c64 and c128 (the bench's headline is qft27
c64); rand30: build_random_circuit(30, 20, seed) fused, c64 and c128, plus
the c64-vs-c128 agreement; qft34: QFT-34 c64 (128 GiB) with the GHZ closed
form checked on sampled indices; sdrp54: min-SDRP search (validate.py:280-300)
for 54 qubits x 7 layers at a device budget; hybrid: QFT-n on GHZ through
the hybrid engine (the paper's Fig. 1b path, cli.py:87-98)."""
from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_14969_b200 import _lib  # noqa: E402
from paper_2304_14969_b200.circuit import build_ghz, build_qft, build_random_circuit  # noqa: E402
from paper_2304_14969_b200.executor import compile_circuit  # noqa: E402
from paper_2304_14969_b200.ket import DenseKet  # noqa: E402

PEAK = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6547.2
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
_lib.call("sk_set_stream", 0, stream.cuda_stream)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def time_program(prog, st, reps=5, warm=2):
    for _ in range(warm):
        prog.run(st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        prog.run(st)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), sum(ts) / len(ts)


def fused(name, circ, dtype, layers):
    n = circ.width
    prog = compile_circuit(circ, dtype=dtype)
    st = DenseKet(n, dtype=dtype)
    best, mean = time_program(prog, st)
    esz = 8 if dtype == "c64" else 16
    sweep_bytes = prog.n_sweeps * 2 * esz * (1 << n)
    emit(config=name, dtype=dtype, qubits=n, gates=len(circ.gates), sweeps=prog.n_sweeps, ms=mean, best_ms=best,
         hbm_gbs=sweep_bytes / (mean / 1e3) / 1e9, frac=sweep_bytes / (mean / 1e3) / 1e9 / PEAK,
         gate_layers_per_s=layers / (mean / 1e3), amp_layers_per_s=layers * (1 << n) / (mean / 1e3))
    del st, prog
    torch.cuda.empty_cache()


def qft(n):
    for dtype in ("c64", "c128"):
        fused(f"qft{n}", build_qft(n), dtype, n)


def rand30():
    c = build_random_circuit(30, 20, 1)
    for dtype in ("c64", "c128"):
        fused("rand30x20", c, dtype, 20)
    # fp32 vs fp64 agreement at full size (no CPU oracle at 30q: ~4 h)
    outs = {}
    for dtype in ("c64", "c128"):
        prog = compile_circuit(c, dtype=dtype)
        st = DenseKet(30, dtype=dtype)
        prog.run(st)
        from paper_2304_14969_b200.ket import permute_qubits
        if prog.plan.phys != list(range(30)):
            st = permute_qubits(st, prog.plan.phys)
        outs[dtype] = st
    idx = np.random.default_rng(0).integers(0, 1 << 30, 4096)
    a = np.array([outs["c64"].amplitude(int(i)) for i in idx[:256]])
    b = np.array([outs["c128"].amplitude(int(i)) for i in idx[:256]])
    emit(config="rand30x20", check="c64 vs c128 on 256 sampled amplitudes", max_abs_diff=float(np.max(np.abs(a - b))),
         norm_c64=outs["c64"].norm(), norm_c128=outs["c128"].norm())


def qft34(n=34):
    """QFT-34 c64 (128 GiB resident); input |k> (X on the set bits of k, one
    pass each), output checked against e^{2 pi i jk/N}/sqrt(N) on sampled j."""
    from paper_2304_14969_b200.circuit import gate_matrix
    from paper_2304_14969_b200.ket import permute_qubits  # noqa: F401
    st = DenseKet(n, dtype="c64")
    prog = compile_circuit(build_qft(n), dtype="c64")
    best, mean = time_program(prog, st, reps=3, warm=1)
    sweep_bytes = prog.n_sweeps * 2 * 8 * (1 << n)
    emit(config=f"qft{n}", dtype="c64", qubits=n, sweeps=prog.n_sweeps, ms=mean, best_ms=best,
         hbm_gbs=sweep_bytes / (mean / 1e3) / 1e9, frac=sweep_bytes / (mean / 1e3) / 1e9 / PEAK,
         gate_layers_per_s=n / (mean / 1e3), amp_layers_per_s=n * (1 << n) / (mean / 1e3))
    del st
    torch.cuda.empty_cache()
    k = 0x2D5A5A5A5 & ((1 << n) - 1)
    st = DenseKet(n, dtype="c64")
    for q in range(n):
        if (k >> q) & 1:
            st.apply_1q(q, gate_matrix("x"))
    prog.run(st)
    N = 1 << n
    js = np.random.default_rng(3).integers(0, N, 64)
    err = 0.0
    for j in js:
        # label-order amplitude j lives at the physical index given by the plan's label permutation
        phys = prog.plan.phys
        pj = sum(((int(j) >> lab) & 1) << phys[lab] for lab in range(n))
        want = np.exp(2j * np.pi * ((int(j) * k) % N) / N) / math.sqrt(N)
        err = max(err, abs(st.amplitude(pj) - want))
    emit(config=f"qft{n}", check=f"QFT|k> closed form on 64 sampled amplitudes, k={k}", max_abs_err=err,
         amp_scale=1 / math.sqrt(N))


def sdrp54(budget_log2=31, depth=7, circuits=1):
    from paper_2304_14969_b200.sdrp import min_sdrp_search
    from paper_2304_14969_b200.circuit import derive_seed
    for i in range(circuits):
        seed = derive_seed(0, i)
        trace = []
        t0 = time.perf_counter()
        r = min_sdrp_search(54, depth, seed, 1 << budget_log2, dtype="c64", trace=trace)
        emit(config="sdrp54", depth=depth, circuit=i, budget=1 << budget_log2, feasible=r.feasible, p_min=r.p_min,
             f_model=r.f_model, peak=r.peak_amplitudes, wall_s=time.perf_counter() - t0,
             trace=[(t.p, t.ok, t.f_model, t.peak_amplitudes, round(t.wall_s, 3)) for t in trace])


def sdrp_depths(budget_log2=30, circuits=10, depths=(7, 8, 9, 10)):
    """Paper-style ensemble: per depth, min-SDRP search for
    `circuits` random 54-qubit circuits (validate.py:280-300 semantics) at a
    device budget; mean / median F_model and time per circuit."""
    import statistics
    from paper_2304_14969_b200.circuit import derive_seed
    from paper_2304_14969_b200.sdrp import min_sdrp_search
    for d in depths:
        fs, ps, ts, peaks = [], [], [], []
        for i in range(circuits):
            t0 = time.perf_counter()
            r = min_sdrp_search(54, d, derive_seed(0, i), 1 << budget_log2, dtype="c64")
            ts.append(time.perf_counter() - t0)
            fs.append(r.f_model if r.feasible else 0.0)
            ps.append(r.p_min if r.feasible else None)
            peaks.append(r.peak_amplitudes)
        emit(config="sdrp54_depths", depth=d, circuits=circuits, budget=1 << budget_log2,
             f_model_mean=statistics.mean(fs), f_model_median=statistics.median(fs), f_model_max=max(fs),
             p_min=ps, peak_max=max(peaks), s_per_circuit=statistics.mean(ts))


def hybrid(n=20, reps=3):
    from paper_2304_14969_b200.engine import EngineConfig, HybridState, OptFlags
    for dtype in ("c128", "c64"):
        ts = []
        for rep in range(reps):
            sim = HybridState(n, EngineConfig(mem_budget=1 << 30, dtype=dtype,
                                              optimizations=OptFlags(stabilizer_hybrid=False)))
            sim.apply_circuit(build_ghz(n))
            sim.flush_all()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sim.apply_circuit(build_qft(n))
            sim.flush_all()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        emit(config=f"hybrid_qft{n}_ghz", dtype=dtype, wall_s=sorted(ts)[len(ts) // 2], stats=dict(sim.stats),
             peak=sim.peak_amplitudes)


if __name__ == "__main__":
    want = sys.argv[1:] or ["qft20", "qft27", "rand30", "hybrid"]
    for w in want:
        if w == "qft20":
            qft(20)
        elif w == "qft27":
            qft(27)
        elif w == "rand30":
            rand30()
        elif w == "qft34":
            qft34()
        elif w.startswith("sdrp54"):  # sdrp54[:budget_log2[:circuits]]
            parts = w.split(":")
            sdrp54(int(parts[1]) if len(parts) > 1 else 31, 7, int(parts[2]) if len(parts) > 2 else 1)
        elif w.startswith("sdrpdepths"):  # sdrpdepths[:budget_log2[:circuits]]
            parts = w.split(":")
            sdrp_depths(int(parts[1]) if len(parts) > 1 else 30, int(parts[2]) if len(parts) > 2 else 10)
        elif w.startswith("hybrid"):  # hybrid[:n]
            parts = w.split(":")
            hybrid(int(parts[1]) if len(parts) > 1 else 20, 3 if len(parts) == 1 or int(parts[1]) < 26 else 1)
