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
                 chunk_bytes: int = 1 << 30, schedule: str = "one", overlap: bool = True):
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
        if exchange not in ("alltoall", "pairwise", "host", "host-pairwise"):
            raise ValueError(f"exchange must be 'auto', 'alltoall', 'pairwise', 'host' or 'host-pairwise', "
                             f"got {exchange!r}")
        self.exchange = exchange
        self.overlap = overlap
        self._xstream = None
        nbuf = 2 if (exchange in ("alltoall", "host") and self.G) else 1  # *pairwise: in place, one slab
        self.bufs = [torch.empty(2 << n_local, dtype=real, device=f"cuda:{self.device}") for _ in range(nbuf)]
        self.staging = None
        if exchange.endswith("pairwise") and self.G:
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
        if self.exchange == "host-pairwise":
            blocks = self.state.view(self.world, -1)
            for k in range(1, self.world):
                self._pairwise_step(self.rank ^ k, blocks[self.rank ^ k])
            return
        if self.exchange == "host":
            send = self.state.cpu()
            recv = self.torch.empty_like(send)
            self.dist.all_to_all_single(recv, send, group=self.group)
            self.bufs[1 - self.cur].copy_(recv)
            self.cur = 1 - self.cur
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

    def _blocks_of_last_sweep(self):
        """Tiles per exchange block of the body's last sweep, or None when its
        tiles are not contiguous index ranges (then no overlap)."""
        tb, tiles = C.c_int(), C.c_int64()
        _lib.call("sk_program_sweep_tiles", self.body._h, self.body.n_sweeps - 1, C.byref(tb), C.byref(tiles))
        if tb.value < 0 or tiles.value % self.world:
            return None
        return tiles.value // self.world

    def _post(self, send, dst, recv, src):
        """Async send/recv pair of one block; returns a completion callable
        (device tensors over NCCL; host-staged for gloo)."""
        dist, torch = self.dist, self.torch
        if self.exchange.startswith("host"):
            s_h, r_h = send.cpu(), torch.empty(recv.shape, dtype=recv.dtype)
            works = dist.batch_isend_irecv([dist.P2POp(dist.isend, s_h, dst, self.group),
                                            dist.P2POp(dist.irecv, r_h, src, self.group)])

            def done():
                for w in works:
                    w.wait()
                recv.copy_(r_h)
            return done
        works = dist.batch_isend_irecv([dist.P2POp(dist.isend, send, dst, self.group),
                                        dist.P2POp(dist.irecv, recv, src, self.group)])

        def done():
            for w in works:
                w.wait()  # the current stream waits for NCCL's; the host does not block
        return done

    def _pairwise_step(self, partner: int, blk) -> None:
        """In-place swap of block `blk` with `partner` (its block for this
        rank), chunk by chunk through the staging buffer, stream-ordered on the
        current stream (NCCL: no host wait; gloo: host-staged)."""
        dist, torch = self.dist, self.torch
        csz = self.staging.numel() if self.staging is not None else blk.numel()
        for off in range(0, blk.numel(), csz):
            n = min(csz, blk.numel() - off)
            piece = blk[off:off + n]
            if self.exchange.startswith("host"):
                s_h, r_h = piece.cpu(), torch.empty(n, dtype=piece.dtype)
                for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, s_h, partner, self.group),
                                                 dist.P2POp(dist.irecv, r_h, partner, self.group)]):
                    w.wait()
                piece.copy_(r_h)
                continue
            into = self.staging[:n]  # (NCCL pairwise)
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, piece, partner, self.group),
                                             dist.P2POp(dist.irecv, into, partner, self.group)]):
                w.wait()  # stream wait: the copy below is ordered after the transfer
            piece.copy_(into)

    def _run_overlapped(self, events=None, stream=None) -> bool:
        """One-exchange schedule with the exchange overlapped: the body's last
        sweep (the bottom window: contiguous tiles) runs block by block on the
        compute stream, block b = the amplitudes destined for rank b; when a
        block is written, an exchange stream (waiting on just that block) moves
        it while the next block computes.  All-to-all (double buffer): step k
        sends block rank+k and receives from rank-k.  Pairwise in place (one
        slab, QFT-37 at 128 GiB per GPU): step k swaps block rank^k with the
        partner's.  False when the geometry does not allow it."""
        if not (self.overlap and self.G):
            return False
        K = self._blocks_of_last_sweep()
        if K is None:
            return False
        torch = self.torch
        W, r, nb = self.world, self.rank, self.body.n_sweeps
        pairwise = self.exchange.endswith("pairwise")
        comp = torch.cuda.current_stream()  # libshardcu is bound to it
        if self._xstream is None:
            self._xstream = torch.cuda.Stream(device=self.device)
        xs = self._xstream
        _lib.call("sk_rebind", self._h, self.state.data_ptr())
        if events is not None:
            events[0].record(stream)
        for i in range(nb - 1):
            _lib.call("sk_program_run", self._h, self.body._h, i, 1)
            if events is not None:
                events[i + 1].record(stream)
        src_blocks = self.state.view(W, -1)
        dst_blocks = None if pairwise else self.bufs[1 - self.cur].view(W, -1)
        order = [r ^ k for k in range(1, W)] + [r] if pairwise else [(r + k) % W for k in range(W)]
        pending = []
        for b in order:
            _lib.call("sk_program_run_tiles", self._h, self.body._h, nb - 1, b * K, (b + 1) * K)
            if b == r:
                if not pairwise:
                    dst_blocks[r].copy_(src_blocks[r])  # the own block stays (compute stream)
                continue
            ev = torch.cuda.Event()
            ev.record(comp)
            xs.wait_event(ev)
            with torch.cuda.stream(xs):
                if pairwise:
                    self._pairwise_step(b, src_blocks[b])
                else:
                    src = (2 * r - b) % W  # step k = b - r: receive from rank - k
                    pending.append(self._post(src_blocks[b], b, dst_blocks[src], src))
        if events is not None:
            events[nb].record(stream)
        with torch.cuda.stream(xs):
            for done in pending:
                done()
        comp.wait_stream(xs)
        if not pairwise:
            self.cur = 1 - self.cur
        _lib.call("sk_rebind", self._h, self.state.data_ptr())
        _lib.call("sk_program_run", self._h, self.tail._h, 0, -1)
        return True

    def run(self, events=None, stream=None):
        """One sharded QFT on this rank's slab (stream-ordered on the current
        torch stream; libshardcu must be bound to it).  `events` (n_sweeps+1
        CUDA events) bracket the body's fused sweeps for per-launch timing."""
        if self.schedule == "one":
            if self._run_overlapped(events, stream):
                return
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


# ---------------------------------------------------------------------------
# General sharded circuits ("a non-diagonal gate on a global
# qubit needs a global<->local bit swap"; the QFT above is its specialisation)
# ---------------------------------------------------------------------------
def _is_diag(m) -> bool:
    return m[0, 1] == 0 and m[1, 0] == 0


class ShardedState:
    """An n-qubit state vector sharded over W = 2^G ranks by G global bits,
    one process per GPU (torch.distributed: NCCL on the box, gloo with
    host-staged exchanges in the multi-process tests).

    `layout[label]` is the physical bit of logical qubit `label`: bits below
    n_local are local index bits of every rank's slab, bit n_local + i is bit
    i of the rank.  `run(circuit)` executes a gate list:

      * SWAPs are label permutations (engine.py:525-535);
      * gates on local bits are planned by fusion.py into fused sweeps
        (k_sweep / k_qft) on this rank's slab;
      * a control on a global bit is a rank predicate: the gate is dropped on
        ranks whose bit mismatches and loses the control elsewhere;
      * a diagonal gate whose target is global is a rank constant: a phase on
        the slab (or, with local controls, a controlled phase on one of them);
      * a non-diagonal gate on a global qubit first swaps that global bit with
        the local bit whose qubit is needed again furthest in the future
        (Belady): partner ranks (rank ^ 2^i) exchange the half of their slab
        whose local bit disagrees with their rank bit — one NVLink transfer
        of half a slab per rank, chunked through a staging buffer.
    Rank 0 starts in |0...0>."""

    def __init__(self, n: int, dtype: str = "c64", group=None, exchange: str = "auto",
                 chunk_bytes: int = 1 << 30):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.G = self.world.bit_length() - 1
        if (1 << self.G) != self.world:
            raise ValueError(f"world size must be a power of two, got {self.world}")
        self.n, self.dtype = n, dtype
        self.n_local = n - self.G
        if self.n_local < fusion.GEOMETRY[dtype]["nreg"] + 1:
            raise ValueError(f"need more than {fusion.GEOMETRY[dtype]['nreg']} local qubits, got {self.n_local}")
        if exchange == "auto":
            exchange = "nccl" if dist.is_initialized() and dist.get_backend(group) == "nccl" else "host"
        if exchange not in ("nccl", "host"):
            raise ValueError(f"exchange must be 'auto', 'nccl' or 'host', got {exchange!r}")
        self.exchange = exchange
        self.device = torch.cuda.current_device()
        self.cplx = torch.complex64 if dtype == "c64" else torch.complex128
        self.slab = torch.zeros(1 << self.n_local, dtype=self.cplx, device=f"cuda:{self.device}")
        if self.rank == 0:
            self.slab[0] = 1.0
        self.chunk_elems = max(1, chunk_bytes // self.slab.element_size())
        self.layout = list(range(n))
        self.exchanges = 0
        self.exchange_bytes = 0
        h = C.c_void_p()
        _lib.call("sk_wrap", self.n_local, _lib.DTYPES[dtype], self.device,
                  torch.view_as_real(self.slab).data_ptr(), C.byref(h))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.sk_destroy(h)

    # ---- planning ------------------------------------------------------------------
    def _rank_bit(self, phys: int) -> int:
        return (self.rank >> (phys - self.n_local)) & 1

    def _flush(self, ops: list) -> None:
        """Run the pending local ops as fused sweeps and empty the list."""
        if not ops:
            return
        plan = fusion.plan_ops(fusion.merge_1q(fusion.fuse_diagonal_runs(list(ops))), self.n_local, self.dtype)
        ops.clear()
        from .executor import Program
        Program(plan, self.device).run_handle(self._h)

    def _victim(self, nd_target, start: int, busy: set[int]) -> int:
        """Local bit whose qubit's next non-diagonal use lies furthest ahead
        (nd_target[k] = label acted on non-diagonally by gate k, else -1)."""
        nxt = {}
        for k in range(start, len(nd_target)):
            lab = nd_target[k]
            if lab >= 0 and lab not in nxt:
                nxt[lab] = k
        best, best_at = None, -1
        for lab in range(self.n):
            p = self.layout[lab]
            if p >= self.n_local or p in busy:
                continue
            at = nxt.get(lab, len(nd_target) + 1)
            if at > best_at:
                best, best_at = p, at
        return best

    def _swap_bits(self, g: int, loc: int) -> None:
        """Exchange global bit g with local bit loc (relabel + half-slab transfer)."""
        i = g - self.n_local
        b = (self.rank >> i) & 1
        partner = self.rank ^ (1 << i)
        # elements whose local bit `loc` disagrees with the rank bit move to the partner
        view = self.slab.view(-1, 2, 1 << loc)[:, 1 - b, :]
        flat_rows = view.shape[0]
        rows_per = max(1, self.chunk_elems // view.shape[1])
        for r0 in range(0, flat_rows, rows_per):
            part = view[r0:r0 + rows_per]
            send = part.contiguous()
            recv = self.torch.empty_like(send)
            if self.exchange == "host":
                s_h, r_h = self.torch.view_as_real(send).cpu(), self.torch.empty(send.shape + (2,), dtype=send.real.dtype)
                ops = [self.dist.P2POp(self.dist.isend, s_h, partner, self.group),
                       self.dist.P2POp(self.dist.irecv, r_h, partner, self.group)]
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()
                recv.copy_(self.torch.view_as_complex(r_h))
            else:
                ops = [self.dist.P2POp(self.dist.isend, send, partner, self.group),
                       self.dist.P2POp(self.dist.irecv, recv, partner, self.group)]
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()
            part.copy_(recv)
            self.exchange_bytes += send.numel() * send.element_size()
        self.exchanges += 1
        lg = self.layout.index(g)
        ll = self.layout.index(loc)
        self.layout[lg], self.layout[ll] = loc, g

    def run(self, circuit) -> None:
        gates = list(circuit.gates)
        nd_target = [-1 if g.name in ("swap", "m") or _is_diag(gate_matrix(g.name, g.params)) else g.targets[0]
                     for g in gates]
        ops: list[fusion.Op] = []
        for k, g in enumerate(gates):
            if g.name == "m":
                raise ValueError("measurement gates are not supported on sharded states")
            if g.name == "swap":
                a, b = g.targets
                self.layout[a], self.layout[b] = self.layout[b], self.layout[a]
                continue
            m = gate_matrix(g.name, g.params)
            diag = _is_diag(m)
            if diag and m[0, 0] == 1 and m[1, 1] == 1:
                continue
            # controls on global bits are rank predicates
            live, cmask, cval = True, 0, 0
            local_ctrls = []
            for c, pol in zip(g.controls, g.polarity):
                p = self.layout[c]
                if p >= self.n_local:
                    if self._rank_bit(p) != pol:
                        live = False
                else:
                    cmask |= 1 << p
                    cval |= (1 << p) if pol else 0
                    local_ctrls.append((p, pol))
            t = self.layout[g.targets[0]]
            if t >= self.n_local and not diag:  # bring the target home first
                self._flush(ops)
                busy = {self.layout[c] for c in g.controls}
                self._swap_bits(t, self._victim(nd_target, k + 1, busy))
                t = self.layout[g.targets[0]]
                cmask = cval = 0
                local_ctrls = []
                live = True
                for c, pol in zip(g.controls, g.polarity):  # re-resolve: a control may have moved
                    p = self.layout[c]
                    if p >= self.n_local:
                        live = live and self._rank_bit(p) == pol
                    else:
                        cmask |= 1 << p
                        cval |= (1 << p) if pol else 0
                        local_ctrls.append((p, pol))
            if not live:
                continue
            if t >= self.n_local:  # diagonal on a global target: a rank constant
                d = m[1, 1] if self._rank_bit(t) else m[0, 0]
                if local_ctrls:
                    (p0, pol0), rest = local_ctrls[0], local_ctrls[1:]
                    dm = np.array([[1, 0], [0, d]] if pol0 else [[d, 0], [0, 1]], dtype=complex)
                    rm = rv = 0
                    for p, pol in rest:
                        rm |= 1 << p
                        rv |= (1 << p) if pol else 0
                    ops.append(fusion.Op(fusion.DIAG, p0, fusion._m8(dm), rm, rv))
                else:
                    ops.append(fusion.Op(fusion.DIAG, 0, fusion._m8(np.diag([d, d]))))
                continue
            ops.append(fusion.Op(fusion.DIAG if diag else fusion.MAT, t, fusion._m8(m), cmask, cval))
        self._flush(ops)

    # ---- observables (AllReduce of local reductions) ---------------------------------
    def norm2(self) -> float:
        out = C.c_double()
        _lib.call("sk_norm2", self._h, C.byref(out))
        return self._allreduce(out.value)

    def probability(self, label: int, outcome: int) -> float:
        p = self.layout[label]
        if p >= self.n_local:
            mine = 0.0
            if self._rank_bit(p) == outcome:
                out = C.c_double()
                _lib.call("sk_norm2", self._h, C.byref(out))
                mine = out.value
            return self._allreduce(mine)
        sums = (C.c_double * 4)()
        _lib.call("sk_bloch_sums", self._h, p, sums)
        return self._allreduce(sums[3] if outcome else sums[2])

    def _allreduce(self, x: float) -> float:
        if self.world == 1:
            return float(x)
        dev = "cpu" if self.exchange == "host" else f"cuda:{self.device}"
        t = self.torch.tensor([x], dtype=self.torch.float64, device=dev)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())

    def gather(self) -> np.ndarray | None:
        """The global state in label order on rank 0 (tests / read-out)."""
        mine = self.torch.view_as_real(self.slab).cpu().double().contiguous()
        if self.world == 1:
            slabs = [mine]
        else:
            slabs = [self.torch.empty_like(mine) for _ in range(self.world)] if self.rank == 0 else None
            self.dist.gather(mine, slabs, dst=0, group=self.group)
            if self.rank != 0:
                return None
        phys_state = np.concatenate([self.torch.view_as_complex(s).numpy() for s in slabs])  # index = rank<<nl | local
        idx = np.arange(1 << self.n, dtype=np.int64)
        src = np.zeros_like(idx)
        for lab in range(self.n):  # label-order index bit lab lives at physical bit layout[lab]
            src |= ((idx >> lab) & 1) << self.layout[lab]
        return phys_state[src]
