"""Benchmark: exact QFT on 27 qubits (BASELINE.json configs[1]) on B200.

Metric (BASELINE.json "QFT sec & HBM GB/s"): QFT amplitude-layer updates
per second = (QFT layers x amplitudes) / time, whole job over all ranks (one
layer = H(j) plus its controlled-phase fan; work-normalised so weak scaling
reads directly); the line also carries the QFT seconds, the gate-layers/s
and the HBM GB/s of the fused sweeps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1: a step is one full QFT-27 on a resident random normalised state in the
reference's complex128 arithmetic (2 GiB; `--dtype c64` for fp32 storage,
which is also timed and reported under `extra`), SWAPs as label permutations
like the reference engine (engine.py:525-535).
N>1 (torchrun): BASELINE D4, fp32 only: QFT-(34+log2 N) with 2^34 amplitudes
(128 GiB) per GPU, sharded by global qubits, one in-place NCCL exchange per
QFT (distributed.ShardedQFT).
`e2e` repeats the N=1 step through the C ABI with pinned host buffers (copies
inside the timing); `e2e_dropin` through the drop-in Python API
(dense_reference(build_qft(27), initial=DenseKet(27, x)).amps on a
complex128 numpy array).
`--impl reference` times the reference's own CPU DenseKet (shardsim.ket from
baseline/_ref, else the oracle port) on layer-equivalent slices of the same
QFT-27 kernel list, cycling through every layer.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_QUBITS = 27
D4_QUBITS_PER_GPU = 34  # BASELINE D4: 2^34 c64 amplitudes (128 GiB) per GPU -> QFT-35/36/37 at N = 2/4/8
PEAKS = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
CPP_CORES = 1  # the reference's NumPy ufuncs are single-threaded


# ---------------------------------------------------------------------------
# CPU reference path: the reference's own DenseKet (shardsim.ket) from
# baseline/_ref when it is installed there, else the oracle port of it
# ---------------------------------------------------------------------------
def reference_ket_class():
    """(DenseKet class, kind, where): the unmodified reference package
    installed by scripts/install_reference.sh into baseline/_ref (kind
    "reference"), else the oracle's kernel-identical NumPy port (kind "port")."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "shardsim" / "ket.py").exists():
        sys.path.insert(0, str(ref))
        try:
            sys.dont_write_bytecode = True
            from shardsim.ket import DenseKet as RefKet
            return RefKet, "reference", "shardsim.ket.DenseKet (baseline/_ref, unmodified reference package)"
        except Exception:
            pass
        finally:
            sys.path.remove(str(ref))

    import numpy as np

    from oracle import ket_oracle as O

    class PortKet:  # the oracle's NumPy restatement of ket.py:128-164, same call shape
        def __init__(self, width, amps):
            self.amps = np.ascontiguousarray(amps, dtype=complex)

        def apply_1q(self, q, m):
            O.apply_1q(self.amps, q, m)

        def apply_controlled(self, controls, polarity, target, m):
            O.apply_controlled(self.amps, controls, polarity, target, m)

    return PortKet, "port", "oracle/ket_oracle.py (NumPy port of ket.py:128-164)"


def qft_kernel_list(n: int):
    """The reference's QFT-n kernel sequence (circuit.py build_qft; validate.py:97-110 loop body):
    for j = n-1 .. 0: H(j), then CP(pi/2^k) from qubit j-k onto j for k = 1..j.  SWAPs are
    label swaps (engine.py:525-535), as in our arm.  n + n(n-1)/2 kernels = n "layers"."""
    out = []
    for j in range(n - 1, -1, -1):
        out.append(("h", j, None))
        for k in range(1, j + 1):
            out.append(("cp", j, (j - k, math.pi / (1 << k))))
    return out


class CpuQftSampler:
    """Times the reference's CPU QFT-n kernels in slices of one layer-equivalent:
    the n + C(n,2) kernels split into n equal consecutive slices (slice s = kernels
    [s*L, (s+1)*L), L = (n+1)/2 for odd n), so slices cycle through every layer,
    every target and every control distance; n slices = one whole QFT."""

    def __init__(self, n: int, seed: int = 1234):
        import numpy as np

        from paper_2304_14969_b200.circuit import gate_matrix

        self.n = n
        self.cls, self.kind, self.where = reference_ket_class()
        rng = np.random.default_rng(seed)
        x = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        x /= np.linalg.norm(x)
        self.ket = self.cls(n, x)
        del x
        self.kernels = qft_kernel_list(n)
        self.per_slice = len(self.kernels) // n  # (n+1)/2 for odd n: exact
        self.H = gate_matrix("h")
        self.gm = gate_matrix

    def run_slice(self, s: int) -> float:
        s %= self.n
        t0 = time.perf_counter()
        for kind, j, extra in self.kernels[s * self.per_slice:(s + 1) * self.per_slice]:
            if kind == "h":
                self.ket.apply_1q(j, self.H)
            else:
                c, theta = extra
                self.ket.apply_controlled((c,), (1,), j, self.gm("p", (theta,)))
        return time.perf_counter() - t0

    def sample_desc(self, slices) -> str:
        return (f"{len(slices)} of the {self.n} layer-equivalent slices of the QFT-{self.n} kernel list "
                f"(slices {list(slices)}; each {self.per_slice} of its {len(self.kernels)} H/CP kernels) on a "
                f"complex128 2^{self.n} state through {self.where}; 1 thread (NumPy ufuncs are single-threaded); "
                f"SWAPs as label swaps")


def cpu_baseline(n: int):
    """Bounded (~15 s) sample for the cpu_baseline key: every third slice."""
    samp = CpuQftSampler(n)
    slices = list(range(0, n, 3))
    times = [samp.run_slice(s) for s in slices]
    t_layer = statistics.mean(times)
    return {"value": float(1 << n) / t_layer, "unit": "amp-layers/s", "cores": CPP_CORES,
            "host_cores": os.cpu_count(), "kind": samp.kind, "qft_sec": n * t_layer,
            "sample": samp.sample_desc(slices)}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    n_job = (args.qubits or (N_QUBITS if world == 1 else D4_QUBITS_PER_GPU)) + (world.bit_length() - 1)
    n = min(n_job, N_QUBITS)  # a complex128 CPU state above 2^27 (2 GiB) is not a bounded sample
    samp = CpuQftSampler(n)
    times = []
    for i in range(args.warmup + args.steps):
        dt = samp.run_slice(i)
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    value = float(1 << n) / t  # one layer-equivalent over 2^n amplitudes per step
    timed = [i % n for i in range(args.warmup, args.warmup + args.steps)]
    line = {"metric": "QFT amplitude-layer updates/s", "value": value, "unit": "amp-layers/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"exact QFT on {n_job} qubits; reference CPU path"
                                   + ("" if n == n_job else f", sampled at width {n} (time per amplitude-layer is "
                                                            f"width-independent: every kernel is one pass over 2^n)"),
                       "qubits": n_job, "sample_qubits": n, "input": "random normalised complex128 state (seeded, host)",
                       "step": f"one layer-equivalent slice ({samp.per_slice} kernels) of the QFT-{n} kernel list; "
                               f"steps cycle through all {n} slices"},
            "qft_sec": n_job * t * 2.0 ** (n_job - n),
            "cpu_baseline": {"value": value, "unit": "amp-layers/s", "cores": CPP_CORES,
                             "host_cores": os.cpu_count(), "kind": samp.kind,
                             "sample": samp.sample_desc(sorted(set(timed)))},
            "e2e": {"value": value, "unit": "amp-layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (NVML, in-process) for the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
_SASS_KEY = None


def _start_sass_key():
    """Hash the k_qft SASS (cuobjdump, ~20 s) on a host thread while the GPU
    work runs."""
    global _SASS_KEY
    if _SASS_KEY is None:
        from concurrent.futures import ThreadPoolExecutor

        from paper_2304_14969_b200 import _build

        _SASS_KEY = ThreadPoolExecutor(max_workers=1).submit(_build.kernel_sass_sha256, "k_qft")


def _so_sha256() -> str | None:
    """SASS hash of the built library's k_qft kernels (what the committed
    ncu capture measured; file and fatbin bytes differ between identical
    builds)."""
    _start_sass_key()
    try:
        return _SASS_KEY.result(timeout=300)
    except Exception:
        return None


def ncu_traffic(dtype: str, n: int):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full summary, used ONLY when that capture was taken of this exact
    k_qft kernel code (sha256 of their SASS) and workload; else None."""
    prof = ROOT / "profiles" / "ncu_summary.json"
    if not prof.exists():
        return None
    try:
        d = json.loads(prof.read_text())
        entry = d.get("captures", {}).get(f"qft{n}_{dtype}")
        if entry and d.get("kqft_sass_sha256") == _so_sha256():
            return entry.get("dram_bytes_per_launch")
    except Exception:
        return None
    return None


def run_ours(args, rank: int, world: int):
    import numpy as np
    import torch

    from paper_2304_14969_b200 import _lib
    from paper_2304_14969_b200.distributed import ShardedQFT
    from paper_2304_14969_b200.ket import set_default_device

    dev = int(os.environ.get("LOCAL_RANK", 0))
    if int(os.environ.get("RANK", 0)) == 0:
        _start_sass_key()
    torch.cuda.set_device(dev)
    set_default_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    stream = torch.cuda.Stream(device=dev)  # one stream: library kernels, NCCL ordering and the timing events
    torch.cuda.set_stream(stream)
    _lib.call("sk_set_stream", dev, stream.cuda_stream)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n_local = args.qubits if args.qubits else (N_QUBITS if world == 1 else D4_QUBITS_PER_GPU)

    def resident(dtype: str, steps: int, sample_clocks: bool):
        """Time `steps` full QFTs on a resident random state (device-generated)."""
        sq = ShardedQFT(n_local, dtype)  # world == 1: the plain single-GPU QFT-n program
        g = torch.Generator(device=f"cuda:{dev}").manual_seed(1234 + rank)
        sq.state.normal_(generator=g)  # in place: no second slab at 34 qubits
        sq.state.div_(torch.linalg.vector_norm(sq.state) * math.sqrt(world))
        torch.cuda.synchronize()
        nb = sq.body.n_sweeps
        for _ in range(args.warmup):
            sq.run(None, stream)
        barrier()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nb + 1)] for _ in range(steps)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = ClockSampler(dev) if sample_clocks else None
        if clk:
            clk.__enter__()
        barrier()
        start.record(stream)
        for k in range(steps):
            sq.run(evs[k], stream)
        stop.record(stream)
        torch.cuda.synchronize()
        if clk:
            if len(clk.samples) < 20:  # keep sampling a little so short regions still get clock readings
                t_end = time.time() + 0.2
                while time.time() < t_end:
                    sq.run(None, stream)
                torch.cuda.synchronize()
            clk.__exit__()
        ms = max_over_ranks(start.elapsed_time(stop)) / steps
        launch_ms = [evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(steps) for i in range(nb)]
        return sq, ms, launch_ms, clk

    dtype = args.dtype
    sq, ms_per_step, launch_ms, clk = resident(dtype, args.steps, True)
    n, G, nb = sq.n, sq.G, sq.body.n_sweeps
    elem = 8 if dtype == "c64" else 16
    slab_bytes = (1 << n_local) * elem
    real = torch.float32 if dtype == "c64" else torch.float64
    amp_layers = n * float(1 << n)  # n QFT layers over 2^n amplitudes, whole job
    value = amp_layers / (ms_per_step / 1e3)
    avg_launch = statistics.mean(launch_ms)
    per_launch_bytes = sq.body.bytes_per_sweep()
    achieved_gbs = per_launch_bytes / (avg_launch / 1e3) / 1e9

    # ---- e2e (1): the C ABI with pinned host buffers ----------------------
    # Every step: pinned host input -> device (sk_upload_native), the QFT
    # program(s), device -> pinned host output.  At N=1 the steps are
    # double-buffered over two device slabs and two streams, so step k's
    # device->host copy overlaps step k+1's host->device copy and QFT (the
    # copy engines are full duplex); at N>1 the sharded step's NCCL exchanges
    # keep it on one stream.
    e2e_ms, e2e_path = None, "skipped: slab > 4 GiB (two pinned host copies per rank)"
    if slab_bytes <= (4 << 30):
        host_in = [torch.empty(2 << n_local, dtype=real, pin_memory=True) for _ in range(2)]
        for h in host_in:
            h.copy_(sq.state)
        host_out = [torch.empty(2 << n_local, dtype=real, pin_memory=True) for _ in range(2)]
        pipelined = world == 1
        slabs = [sq.state, torch.empty_like(sq.state)] if pipelined else [sq.state]
        streams = [stream, torch.cuda.Stream(device=dev)] if pipelined else [stream]

        def e2e_step(k):
            i = k % len(slabs)
            if pipelined:
                _lib.call("sk_set_stream", dev, streams[i].cuda_stream)
                _lib.call("sk_rebind", sq._h, slabs[i].data_ptr())
                _lib.call("sk_upload_native", sq._h, host_in[i].data_ptr(), 1 << n_local)
                _lib.call("sk_program_run", sq._h, sq.body._h, 0, -1)
                _lib.call("sk_download_native_async", sq._h, host_out[i].data_ptr(), 1 << n_local)
            else:
                _lib.call("sk_rebind", sq._h, sq.state.data_ptr())
                _lib.call("sk_upload_native", sq._h, host_in[0].data_ptr(), 1 << n_local)
                sq.run(None, stream)
                _lib.call("sk_rebind", sq._h, sq.state.data_ptr())
                _lib.call("sk_download_native", sq._h, host_out[0].data_ptr(), 1 << n_local)

        for k in range(2):
            e2e_step(k)
        torch.cuda.synchronize()
        e2e_steps = max(4, min(args.steps, 10))
        barrier()
        e_start, e_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        streams[-1].wait_stream(stream)
        for k in range(e2e_steps):
            e2e_step(k)
        if pipelined:
            _lib.call("sk_set_stream", dev, stream.cuda_stream)
            stream.wait_stream(streams[1])
        e_stop.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e_start.elapsed_time(e_stop) / e2e_steps)
        e2e_path = ("sk_upload_native + QFT program + sk_download_native_async, double-buffered over 2 slabs "
                    "and 2 streams" if pipelined else "sk_upload_native + QFT program(s) + sk_download_native")
        _lib.call("sk_rebind", sq._h, sq.state.data_ptr())
        del host_in, host_out, slabs

    # ---- e2e (2): the drop-in Python API on complex128 host arrays ---------
    # What a reference user calls: dense_reference(build_qft(n), initial=DenseKet(n, x)).amps
    # (validate.py:83-111 signature): upload + plan + fused sweeps + label-order
    # permutation + download, wall-clock timed, synchronised at both ends.
    dropin = None
    if world == 1 and slab_bytes <= (4 << 30) and not args.no_dropin:
        from paper_2304_14969_b200.circuit import build_qft
        from paper_2304_14969_b200.executor import dense_reference
        from paper_2304_14969_b200.ket import DenseKet

        rng = np.random.default_rng(5)
        x = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        x /= np.linalg.norm(x)
        circ = build_qft(n)
        for _ in range(1):
            y = dense_reference(circ, initial=DenseKet(n, x, dtype=dtype)).amps
        torch.cuda.synchronize()
        d_steps = 3
        t0 = time.perf_counter()
        for _ in range(d_steps):
            y = dense_reference(circ, initial=DenseKet(n, x, dtype=dtype)).amps
        torch.cuda.synchronize()
        d_ms = (time.perf_counter() - t0) * 1e3 / d_steps
        dropin = {"value": amp_layers / (d_ms / 1e3), "unit": "amp-layers/s", "ms_per_step": d_ms,
                  "h2d_bytes_per_step": x.nbytes, "d2h_bytes_per_step": y.nbytes,
                  "path": f"paper_2304_14969_b200.executor.dense_reference(build_qft({n}), "
                          f"initial=DenseKet({n}, x, dtype='{dtype}')).amps on a complex128 numpy array "
                          f"(pageable host memory; upload, plan, {nb} sweeps, label-order permutation, download)",
                  "steps": d_steps}
        del x, y

    # ---- the other precision, resident, for reference ----------------------
    extra = {}
    if world == 1 and not args.no_extra:
        other = "c64" if dtype == "c128" else "c128"
        del sq
        torch.cuda.empty_cache()
        sq2, ms2, launch2, _ = resident(other, args.steps, False)
        a2 = statistics.mean(launch2)
        b2 = sq2.body.bytes_per_sweep()
        extra[other] = {"ms_per_step": ms2, "value": amp_layers / (ms2 / 1e3), "unit": "amp-layers/s",
                        "avg_launch_ms": a2, "launch_gbs": b2 / (a2 / 1e3) / 1e9,
                        "roofline_frac": b2 / (a2 / 1e3) / 1e9 / PEAKS.get("hbm_gbs", 6650.0),
                        "sweeps_per_qft": sq2.launches()}
        sq = sq2

    peak = PEAKS.get("hbm_gbs", 6650.0)
    if rank == 0:
        cpu = cpu_baseline(n_local) if (world == 1 and not args.no_cpu) else None
        line = {
            "metric": "QFT amplitude-layer updates/s", "value": value, "unit": "amp-layers/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": f"exact QFT on {n} qubits ({n_local} per GPU x {world} GPU"
                                   f"{'s, global-qubit sharded' if world > 1 else ''})"
                                   + ("; BASELINE configs[1]" if world == 1 and n == 27 else
                                      "; BASELINE configs[3]" if world > 1 else ""),
                       "qubits": n, "qubits_per_gpu": n_local, "state_bytes_per_gpu": slab_bytes,
                       "input": "random normalised state, device-generated",
                       "l2": f"state ({slab_bytes / 2**30:g} GiB per GPU) > L2 (126 MB): no flush needed",
                       "swaps": "label permutations (engine.py:525-535)",
                       "parallelism": f"global-qubit sharding over {world} GPUs (one-exchange schedule: "
                                      f"1 NCCL all-to-all per QFT, {sq.exchange})" if world > 1 else "single GPU"},
            "qft_sec": ms_per_step / 1e3,
            "qft_qubits": n,
            "gate_layers_per_s": n / (ms_per_step / 1e3),
            "hbm_gbs": nb * per_launch_bytes / (ms_per_step / 1e3) / 1e9,
            "sweeps_per_qft": nb + (1 if world > 1 else 0),
            "exchange_bytes_per_gpu": sq.exchange_bytes(),
            "unfused_bytes_per_qft_per_gpu": 2 * elem * (n * (1 << n_local) + (n * (n - 1) // 2) * (1 << (n_local - 1))),
            "gpu_launches": args.steps * (nb + (1 if world > 1 else 0)),
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                         "frac": achieved_gbs / peak, "traffic": ncu_traffic(dtype, n_local),
                         "kernel": f"k_qft<{'float' if dtype == 'c64' else 'double'},4,NS>",
                         "algorithmic_bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_launch,
                         "launches_per_step": nb,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if PEAKS else "fallback (B200_PROFILING.md)"},
            "clocks": clk.summary() if clk else None,
            "e2e": {"value": amp_layers / (e2e_ms / 1e3) if e2e_ms else None, "unit": "amp-layers/s",
                    "h2d_bytes_per_step": slab_bytes * world, "d2h_bytes_per_step": slab_bytes * world,
                    "ms_per_step": e2e_ms, "path": e2e_path},
            "e2e_dropin": dropin,
            "extra": extra,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--qubits", type=int, default=0,
                    help=f"qubits per GPU (default {N_QUBITS} at N=1, {D4_QUBITS_PER_GPU} per GPU at N>1: BASELINE D4)")
    ap.add_argument("--dtype", default=None, choices=["c64", "c128"],
                    help="default c128 = the reference's complex128 arithmetic (ket.py:77,82) at N=1; "
                         "c64 at N>1 (BASELINE D4 is fp32: a c128 2^34 slab is 256 GiB)")
    ap.add_argument("--no-dropin", action="store_true", help="skip the drop-in API e2e leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the other-precision resident line")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if "RANK" in os.environ else 1))
    if args.dtype is None:
        args.dtype = "c128" if world == 1 else "c64"
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
