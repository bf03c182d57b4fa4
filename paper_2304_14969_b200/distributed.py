"""Global-qubit sharding of the QFT over 2^G ranks.

An n-qubit state is split by its top G index bits ("global" qubits): rank r
holds the 2^(n-G) amplitudes whose top bits equal r.  The reference has no
distributed path; this is the B200-native extension that makes QFT-37 fit on
8 GPUs.  The QFT needs exactly two exchanges:

  A. all-to-all swapping the global bits [n-G, n) with the top local bits
     [n-2G, n-G) (equal 2^(n-2G)-amplitude blocks: block b of rank r goes to
     rank b, slot r) — the top G logical qubits become local;
  1. one generic fused sweep applies QFT layers j = n-1 .. n-G.  Their CP fans
     split into a local RAMP over bits [0, n-2G), a local RAMP over the moved
     top qubits, and a phase that is a rank constant (the fan's contribution
     from the now-global logical qubits [n-2G, n-G));
  B. the same all-to-all again: the layout is the identity once more;
  2. layers j < n-G have all their controls local: each rank runs exactly the
     (n-G)-qubit QFT body (the FFT-form fused sweeps of fusion.plan_qft).

The QFT's final SWAP layer stays a label permutation (full bit reversal).
Exchanges go through torch.distributed (NCCL over NVLink on the box; gloo in
the CPU tests), on torch buffers wrapped as non-owning sk_state views.

One-exchange schedule (schedule="one", the default).  If instead the rank
holds the LOW G qubits (rank r owns the amplitudes whose index ends in r;
local bit b = qubit b + G), the QFT's first n-G layers (targets n-1..G) are
all local: each rank runs the ordinary (n-G)-qubit FFT-form body with its
phase index shifted to (i << G) | r, which folds the controlled phases from
the G rank-constant qubits into the windows' twiddles
(sk_program_set_phase_index).  One all-to-all then swaps the rank bits with
the top G local bits, and a single fused sweep runs the last G layers on the
moved qubits.  Half the NVLink traffic of the two-exchange schedule for the
same HBM passes.  The result has the high G qubits as rank bits (`one_x_label`
gives the element -> qubit-index map); the bit reversal stays a label swap.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib, fusion
from .circuit import gate_matrix


def layout(n_local: int, world: int) -> tuple[int, int]:
    """(n, G) for `world` ranks of 2^n_local amplitudes each."""
    G = world.bit_length() - 1
    if world < 1 or (1 << G) != world:
        raise ValueError(f"world size must be a power of two, got {world}")
    if G and n_local < 2 * G + 1:
        raise ValueError(f"need n_local >= 2G+1 ({2 * G + 1}) local qubits, got {n_local}")
    return n_local + G, G


def top_layer_ops(n_local: int, G: int, rank: int) -> list[fusion.Op]:
    """Ops (local physical bits) of QFT layers j = n-1..n-G after exchange A."""
    n = n_local + G
    lo2 = n - 2 * G
    ops: list[fusion.Op] = []
    h = fusion._m8(gate_matrix("h"))
    for j in range(n - 1, n - G - 1, -1):
        P = j - G
        ops.append(fusion.Op(fusion.MAT, P, h))
        if lo2 >= 1:  # controls [0, n-2G): local, weights 2^(i-j)
            ops.append(fusion.Op(fusion.RAMP, 0, (2.0 ** -j, 0, 0, 0, 0, 0, 0, 0), 1 << P, 1 << P, nbits=lo2))
        # controls [n-2G, n-G) now sit in the rank bits: a rank-constant phase on P
        theta = sum(math.pi * 2.0 ** (i - j) for i in range(lo2, n - G) if (rank >> (i - lo2)) & 1)
        if theta:
            ops.append(fusion.Op(fusion.DIAG, P, (1.0, 0, 0, 0, 0, 0, math.cos(theta), math.sin(theta))))
        if P - lo2 >= 1:  # controls [n-G, j) moved to local [n-2G, P): weights 2^(p-P)
            ops.append(fusion.Op(fusion.RAMP, lo2, (2.0 ** (lo2 - P), 0, 0, 0, 0, 0, 0, 0), 1 << P, 1 << P,
                                 nbits=P - lo2))
    return ops


def plans(n_local: int, world: int, rank: int, dtype: str = "c64"):
    """(top-layer plan or None, local QFT-body plan) for one rank."""
    n, G = layout(n_local, world)
    body = fusion.plan_qft(n_local, dtype)
    if G == 0:
        return None, body
    top = fusion.plan_ops(top_layer_ops(n_local, G, rank), n_local, dtype)
    return top, body


def tail_ops(n_local: int, G: int) -> list[fusion.Op]:
    """Ops of QFT layers G-1..0 after the exchange of the one-exchange
    schedule: qubit j < G sits at local bit n_local - G + j; its CP fan comes
    only from the moved qubits k < j."""
    from .circuit import Circuit, cp, h
    base = n_local - G
    gates = []
    for j in range(G - 1, -1, -1):
        gates.append(h(base + j))
        for k in range(j - 1, -1, -1):
            gates.append(cp(math.pi / (1 << (j - k)), base + k, base + j))
    ops, _ = fusion.lower(Circuit(n_local, tuple(gates)))
    return fusion.fuse_diagonal_runs(ops)


def plans_one_exchange(n_local: int, world: int, dtype: str = "c64"):
    """(body plan, tail plan or None) of the one-exchange schedule; the body
    runs with phase index (i << G) | rank on every rank."""
    n, G = layout(n_local, world)
    body = fusion.plan_qft(n_local, dtype)
    tail = fusion.plan_ops(tail_ops(n_local, G), n_local, dtype) if G else None
    return body, tail


def one_x_label(n_local: int, G: int) -> np.ndarray:
    """Qubit-order index (before the QFT's final SWAP layer) of element
    (rank s, local l) after the one-exchange schedule, as a flat array over
    s * 2^n_local + l: rank bits = qubits n-G..n-1, local top bits = qubits
    0..G-1, local bits b < n_local - G = qubit b + G."""
    n = n_local + G
    s = np.repeat(np.arange(1 << G, dtype=np.int64), 1 << n_local)
    l = np.tile(np.arange(1 << n_local, dtype=np.int64), 1 << G)
    lo = l & ((1 << (n_local - G)) - 1)
    top = l >> (n_local - G)
    return (s << (n - G)) | (lo << G) | top


def final_order(n: int) -> list[int]:
    """permute_qubits order mapping the physical result to label order (the
    QFT's reversal swaps as a label permutation)."""
    return list(reversed(range(n)))


def exchange_blocks(slabs: list[np.ndarray]) -> list[np.ndarray]:
    """all_to_all_single semantics on equal blocks, for the NumPy emulation:
    out[r] block s = in[s] block r."""
    W = len(slabs)
    blocks = [np.split(s, W) for s in slabs]
    return [np.concatenate([blocks[s][r] for s in range(W)]) for r in range(W)]


def emulate(slabs: list[np.ndarray], dtype: str = "c64") -> list[np.ndarray]:
    """Single-process NumPy emulation of the sharded QFT (all ranks), used by
    the CPU tests to check the plan/exchange logic against the oracle."""
    W = len(slabs)
    n_local = int(slabs[0].size).bit_length() - 1
    n, G = layout(n_local, W)
    cur = [s.copy() for s in slabs]
    if G:
        cur = exchange_blocks(cur)
        for r in range(W):
            top, _ = plans(n_local, W, r, dtype)
            fusion.run_plan_numpy(top, cur[r])
        cur = exchange_blocks(cur)
    for r in range(W):
        _, body = plans(n_local, W, r, dtype)
        fusion.run_plan_numpy(body, cur[r])
    return cur


def pairwise_exchange(dist, buf, staging, world: int, rank: int, group=None) -> None:
    """In-place all_to_all_single on equal blocks (out[r] block s = in[s]
    block r) as W-1 pairwise swaps: at step k rank r swaps its block r^k with
    the partner's block r, chunk by chunk through `staging` (any size).  The
    whole exchange needs one slab plus the staging buffer instead of two
    slabs, which is what lets QFT-37 (2^34 amplitudes = 128 GiB per GPU)
    fit on 8 x 180 GB."""
    blocks = buf.view(world, -1)
    csz = min(staging.numel(), blocks.shape[1])
    for k in range(1, world):
        partner = rank ^ k
        blk = blocks[partner]
        for off in range(0, blk.numel(), csz):
            n = min(csz, blk.numel() - off)
            piece, into = blk[off:off + n], staging[:n]
            ops = [dist.P2POp(dist.isend, piece, partner, group), dist.P2POp(dist.irecv, into, partner, group)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            piece.copy_(into)


def scatter_input(x: np.ndarray, world: int, rank: int, schedule: str = "one") -> np.ndarray:
    """This rank's input slab of the global n-qubit vector x.  schedule "one"
    (the default): the rank holds the LOW G qubits, slab = x[rank::world];
    schedule "two": the rank holds the top G qubits, slab = contiguous block."""
    if schedule == "one":
        return np.ascontiguousarray(x[rank::world])
    return np.ascontiguousarray(np.split(x, world)[rank])


def assemble_output(slabs, n_local: int, G: int, schedule: str = "one") -> np.ndarray:
    """The global QFT output in qubit-index order (before the QFT's final SWAP
    layer, which stays a label permutation: apply final_order(n) for label
    order) from every rank's output slab, rank order."""
    flat = np.concatenate([np.asarray(s) for s in slabs])
    if schedule == "two" or G == 0:
        return flat
    u = np.empty(flat.size, dtype=flat.dtype)
    u[one_x_label(n_local, G)] = flat
    return u


class ShardedQFT:
    """Device execution on one rank: the slab (and, for the double-buffered
    exchange, a second one) as torch buffers wrapped as sk_state views;
    NCCL all_to_all_single or in-place pairwise NCCL send/recv for the
    exchanges; fused sweeps for the local work.

    Layout (it depends on the schedule):
      * schedule="one" (default, one exchange per QFT): input slab of rank r =
        x[r::W] (the rank holds the LOW G qubits); the output has the high G
        qubits as rank bits, element order `one_x_label`.  `scatter_input` /
        `assemble_output` convert to and from global vectors.
      * schedule="two": input and output are contiguous blocks (rank = top G
        qubits), two exchanges per QFT.
    In both, the QFT's final SWAP layer is a label permutation (final_order).

    exchange="auto" picks the double-buffered all-to-all when two slabs fit in
    device memory and the in-place pairwise exchange (one slab + a
    `chunk_bytes` staging buffer) otherwise.  exchange="host" stages the
    all-to-all through host memory, for process groups whose backend cannot
    move device buffers (gloo: the multi-process tests on one GPU)."""

    def __init__(self, n_local: int, dtype: str = "c64", group=None, exchange: str = "auto",
                 chunk_bytes: int = 1 << 30, schedule: str = "one"):
        import torch
        import torch.distributed as dist

        from .executor import Program
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n_local, self.dtype = n_local, dtype
        self.n, self.G = layout(n_local, self.world)
        self.device = torch.cuda.current_device()
        real = torch.float32 if dtype == "c64" else torch.float64
        slab_bytes = (1 << n_local) * (8 if dtype == "c64" else 16)
        if exchange == "auto":
            free, _ = torch.cuda.mem_get_info(self.device)
            exchange = "alltoall" if (self.G == 0 or 2 * slab_bytes + (4 << 30) <= free) else "pairwise"
        if exchange not in ("alltoall", "pairwise", "host"):
            raise ValueError(f"exchange must be 'auto', 'alltoall', 'pairwise' or 'host', got {exchange!r}")
        self.exchange = exchange
        nbuf = 2 if (exchange == "alltoall" and self.G) else 1
        self.bufs = [torch.empty(2 << n_local, dtype=real, device=f"cuda:{self.device}") for _ in range(nbuf)]
        self.staging = None
        if exchange == "pairwise" and self.G:
            n_stage = min((2 << n_local) // self.world, max(2, chunk_bytes // real.itemsize))
            self.staging = torch.empty(n_stage, dtype=real, device=f"cuda:{self.device}")
        self.cur = 0
        h = C.c_void_p()
        _lib.call("sk_wrap", n_local, _lib.DTYPES[dtype], self.device, self.bufs[0].data_ptr(), C.byref(h))
        self._h = h
        if schedule not in ("one", "two"):
            raise ValueError(f"schedule must be 'one' or 'two', got {schedule!r}")
        self.schedule = schedule
        self.top = self.tail = None
        if schedule == "one":
            body, tail = plans_one_exchange(n_local, self.world, dtype)
            self.body = Program(body, self.device)
            if self.G:
                self.body.set_phase_index(self.G, self.rank)
                self.tail = Program(tail, self.device)
        else:
            top, body = plans(n_local, self.world, self.rank, dtype)
            self.top = Program(top, self.device) if top is not None else None
            self.body = Program(body, self.device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.sk_destroy(h)

    @property
    def state(self):
        return self.bufs[self.cur]

    def _exchange(self):
        if self.exchange == "host":
            send = self.state.cpu()
            recv = self.torch.empty_like(send)
            self.dist.all_to_all_single(recv, send, group=self.group)
            self.state.copy_(recv)
            return
        if self.exchange == "pairwise":
            pairwise_exchange(self.dist, self.bufs[0], self.staging, self.world, self.rank, self.group)
            return
        nxt = 1 - self.cur
        self.dist.all_to_all_single(self.bufs[nxt], self.bufs[self.cur], group=self.group)
        self.cur = nxt

    def _run_body(self, events=None, stream=None):
        _lib.call("sk_rebind", self._h, self.state.data_ptr())
        if events is None:
            _lib.call("sk_program_run", self._h, self.body._h, 0, -1)
            return
        events[0].record(stream)
        for i in range(self.body.n_sweeps):
            _lib.call("sk_program_run", self._h, self.body._h, i, 1)
            events[i + 1].record(stream)

    def run(self, events=None, stream=None):
        """One sharded QFT on this rank's slab (stream-ordered on the current
        torch stream; libshardcu must be bound to it).  `events` (n_sweeps+1
        CUDA events) bracket the body's fused sweeps for per-launch timing."""
        if self.schedule == "one":
            self._run_body(events, stream)
            if self.G:
                self._exchange()
                _lib.call("sk_rebind", self._h, self.state.data_ptr())
                _lib.call("sk_program_run", self._h, self.tail._h, 0, -1)
            return
        if self.G:
            self._exchange()
            _lib.call("sk_rebind", self._h, self.state.data_ptr())
            _lib.call("sk_program_run", self._h, self.top._h, 0, -1)
            self._exchange()
        self._run_body(events, stream)

    def launches(self) -> int:
        extra = self.tail if self.schedule == "one" else self.top
        return (extra.n_sweeps if extra else 0) + self.body.n_sweeps

    def exchange_bytes(self) -> int:
        """Bytes each rank sends per QFT (one or two all-to-alls, own block stays)."""
        if not self.G:
            return 0
        elem = 8 if self.dtype == "c64" else 16
        per = (self.world - 1) * ((1 << self.n_local) // self.world) * elem
        return per * (1 if self.schedule == "one" else 2)
