"""Benchmark: exact QFT on 27 qubits (BASELINE.json configs[1]) on B200.

Metric (BASELINE.json "QFT sec & HBM GB/s"): QFT amplitude-layer updates
per second = (QFT layers x amplitudes) / time, whole job over all ranks (one
layer = H(j) plus its controlled-phase fan; work-normalised so weak scaling
reads directly); the line also carries the QFT seconds, the gate-layers/s
and the HBM GB/s of the fused sweeps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one full QFT-27 at N=1 (fp32 amplitudes, 1 GiB, random normalised
input, SWAPs as label permutations like the reference engine) on a resident
state; at N GPUs one QFT-(27+log2 N) sharded by global qubits (1 GiB per GPU,
two NCCL all-to-alls per QFT).
`e2e` repeats it through the public C-ABI entry points with host buffers:
pinned host state -> device, QFT, device -> host, copies inside the timing.
`--impl reference` times the reference's CPU path (the oracle port of its
NumPy kernels, oracle/ket_oracle.py) on the same workload.
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
CPP_CORES = 1  # the reference's NumPy ufuncs are single-threaded


# ---------------------------------------------------------------------------
# CPU reference path (oracle port of the reference's kernels)
# ---------------------------------------------------------------------------
def cpu_layer_sample(n: int, n_cp: int | None = None):
    """Time one 'average' QFT layer of the reference's dense loop at width n:
    one H plus (n-1)/2 controlled phases (QFT-n = n H + C(n,2) CP), complex128,
    through the oracle's kernel-identical NumPy expressions (ket.py:133-164)."""
    import numpy as np

    from oracle import ket_oracle as O
    from paper_2304_14969_b200.circuit import gate_matrix

    n_cp = (n - 1) // 2 if n_cp is None else n_cp
    amps = np.zeros(1 << n, dtype=complex)
    amps[0] = amps[-1] = 2 ** -0.5
    H = gate_matrix("h")
    j = n - 1
    t0 = time.perf_counter()
    O.apply_1q(amps, j, H)
    t1 = time.perf_counter()
    for k in range(1, n_cp + 1):
        O.apply_controlled(amps, (j - k,), (1,), j, gate_matrix("p", (math.pi / (1 << k),)))
    t2 = time.perf_counter()
    return t1 - t0, (t2 - t1) / max(1, n_cp)


def cpu_baseline(n: int):
    m = min(n, 27)  # sample at <= 27 qubits (2 GiB complex128); kernel time scales with 2^n
    t_h, t_cp = cpu_layer_sample(m, 4)
    t_h, t_cp = t_h * 2.0 ** (n - m), t_cp * 2.0 ** (n - m)
    t_qft = n * t_h + (n * (n - 1) // 2) * t_cp
    return {"value": n * float(1 << n) / t_qft, "unit": "amp-layers/s", "cores": CPP_CORES, "kind": "port",
            "qft_sec": t_qft,
            "sample": f"1 H + 4 CP kernels at width {m} (x 2^{n - m} for width {n}) on a complex128 state via the oracle port of the "
                      f"reference's NumPy kernels (ket.py:133-164), 1 thread; extrapolated to the QFT-{n} mix "
                      f"of {n} H + {n * (n - 1) // 2} CP (SWAPs as label swaps, engine.py:525-535)"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    n = args.qubits
    times = []
    for i in range(args.warmup + args.steps):
        t_h, t_cp = cpu_layer_sample(n)
        if i >= args.warmup:
            times.append(t_h + ((n - 1) // 2) * t_cp)
    t = statistics.mean(times)
    value = float(1 << n) / t  # one layer over 2^n amplitudes per step
    line = {"metric": "QFT amplitude-layer updates/s", "value": value, "unit": "amp-layers/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"exact QFT on {n} qubits (BASELINE configs[1]); reference CPU path",
                       "qubits": n, "step": f"one average QFT-{n} layer: 1 H + {(n - 1) // 2} CP kernels"},
            "qft_sec": n * t,
            "cpu_baseline": {"value": value, "unit": "amp-layers/s", "cores": CPP_CORES, "kind": "port",
                             "sample": f"each step = 1 H + {(n - 1) // 2} CP kernels at width {n}, complex128, "
                                       f"oracle port of ket.py:133-164 (NumPy, single-threaded)"},
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
def run_ours(args, rank: int, world: int):
    import torch

    from paper_2304_14969_b200 import _lib
    from paper_2304_14969_b200.distributed import ShardedQFT
    from paper_2304_14969_b200.ket import set_default_device

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    set_default_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    stream = torch.cuda.Stream(device=dev)  # one stream: library kernels, NCCL ordering and the timing events
    torch.cuda.set_stream(stream)
    _lib.call("sk_set_stream", dev, stream.cuda_stream)

    n_local, dtype = args.qubits, args.dtype
    sq = ShardedQFT(n_local, dtype)  # world == 1: the plain single-GPU QFT-n program
    n, G = sq.n, sq.G
    elem = 8 if dtype == "c64" else 16
    slab_bytes = (1 << n_local) * elem
    real = torch.float32 if dtype == "c64" else torch.float64

    # random normalised global state, generated on the device per rank (not timed)
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(1234 + rank)
    sq.state.normal_(generator=g)  # in place: no second slab at 34 qubits
    sq.state.div_(torch.linalg.vector_norm(sq.state) * math.sqrt(world))
    torch.cuda.synchronize()

    body = sq.body
    nb = body.n_sweeps

    def step(evs=None):
        sq.run(evs, stream)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nb + 1)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        barrier()
        start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        stop.record(stream)
        torch.cuda.synchronize()
        if len(clk.samples) < 20:  # keep sampling a little so short regions still get clock readings
            t_end = time.time() + 0.2
            while time.time() < t_end:
                step()
            torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    launch_ms = [evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(args.steps) for i in range(nb)]
    if dist is not None:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    amp_layers = n * float(1 << n)  # n QFT layers over 2^n amplitudes, whole job
    value = amp_layers / (ms_per_step / 1e3)
    avg_launch = statistics.mean(launch_ms)
    per_launch_bytes = body.bytes_per_sweep()
    achieved_gbs = per_launch_bytes / (avg_launch / 1e3) / 1e9

    # ---- e2e through the public API with host buffers --------------------
    # Every step: pinned host input -> device (sk_upload_native), the QFT
    # program(s), device -> pinned host output.  At N=1 the steps are
    # double-buffered over two device slabs and two streams, so step k's
    # device->host copy overlaps step k+1's host->device copy and QFT (the
    # copy engines are full duplex); at N>1 the sharded step's NCCL exchanges
    # keep it on one stream.
    if slab_bytes > (4 << 30):  # e2e pins two host copies of the slab: only at BASELINE's 1 GiB scale
        e2e_ms = None
    host_in = [torch.empty(2 << n_local, dtype=real, pin_memory=True) for _ in range(2)] if slab_bytes <= (4 << 30) \
        else []
    if host_in:
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
                for prog in (body,):
                    _lib.call("sk_program_run", sq._h, prog._h, 0, -1)
                _lib.call("sk_download_native_async", sq._h, host_out[i].data_ptr(), 1 << n_local)
            else:
                _lib.call("sk_rebind", sq._h, sq.state.data_ptr())
                _lib.call("sk_upload_native", sq._h, host_in[0].data_ptr(), 1 << n_local)
                step()
                _lib.call("sk_rebind", sq._h, sq.state.data_ptr())
                _lib.call("sk_download_native", sq._h, out_host.data_ptr(), 1 << n_local)

        out_host = host_out[0]
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
        e2e_ms = e_start.elapsed_time(e_stop) / e2e_steps
        e2e_path = ("sk_upload_native + QFT program + sk_download_native_async, double-buffered over 2 slabs "
                    "and 2 streams" if pipelined else "sk_upload_native + QFT program(s) + sk_download_native")
        if dist is not None:
            t = torch.tensor([e2e_ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
    else:
        e2e_path = "skipped: slab > 4 GiB (two pinned host copies per rank)"

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_sweep")
        except Exception:
            traffic = None

    if rank == 0:
        cpu = cpu_baseline(n_local) if (world == 1 and not args.no_cpu) else None
        line = {
            "metric": "QFT amplitude-layer updates/s", "value": value, "unit": "amp-layers/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": f"exact QFT on {n} qubits ({n_local} per GPU x {world} GPU"
                                   f"{'s, global-qubit sharded' if world > 1 else ''}); BASELINE configs[1] at N=1",
                       "qubits": n, "qubits_per_gpu": n_local, "state_bytes_per_gpu": slab_bytes,
                       "input": "random normalised state, device-generated",
                       "l2": f"state ({slab_bytes / 2**30:g} GiB per GPU) > L2 (126 MB): no flush needed",
                       "swaps": "label permutations (engine.py:525-535)",
                       "parallelism": f"global-qubit sharding over {world} GPUs ({sq.schedule}-exchange schedule: "
                                      f"{1 if sq.schedule == 'one' else 2} NCCL all-to-all(s) per QFT, {sq.exchange})"
                                      if world > 1 else "single GPU"},
            "qft_sec": ms_per_step / 1e3,
            "qft_qubits": n,
            "gate_layers_per_s": n / (ms_per_step / 1e3),
            "hbm_gbs": nb * per_launch_bytes / (ms_per_step / 1e3) / 1e9,
            "sweeps_per_qft": sq.launches(),
            "exchange_bytes_per_gpu": sq.exchange_bytes(),
            "unfused_bytes_per_qft_per_gpu": 2 * elem * (n * (1 << n_local) + (n * (n - 1) // 2) * (1 << (n_local - 1))),
            "gpu_launches": args.steps * sq.launches(),
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                         "frac": achieved_gbs / peak, "traffic": traffic,
                         "kernel": "k_qft<float,4,NS>" if dtype == "c64" else "k_qft<double,3,NS>",
                         "algorithmic_bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_launch,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "clocks": clk.summary(),
            "e2e": {"value": amp_layers / (e2e_ms / 1e3) if e2e_ms else None, "unit": "amp-layers/s",
                    "h2d_bytes_per_step": slab_bytes * world, "d2h_bytes_per_step": slab_bytes * world,
                    "ms_per_step": e2e_ms, "path": e2e_path},
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
    ap.add_argument("--qubits", type=int, default=N_QUBITS)
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if "RANK" in os.environ else 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
