"""Global-qubit sharded QFT (host logic, CPU): the per-rank plans plus the
all-to-all block exchange reproduce the oracle DFT; the exchange semantics
are checked against a real world-size-2/4 gloo all_to_all_single."""
from __future__ import annotations

import os
from pathlib import Path
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ket_oracle as O
from paper_2304_14969_b200 import distributed as D

from conftest import random_state


@pytest.mark.parametrize("world,n_local", [(1, 6), (2, 5), (2, 8), (4, 6), (4, 9), (8, 7)])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_emulated_sharded_qft_equals_dft(rng, world, n_local, dtype):
    n, G = D.layout(n_local, world)
    x = random_state(n, rng)
    slabs = np.split(x.copy(), world)
    out = np.concatenate(D.emulate(slabs, dtype))
    got = O.permute_qubits(out, D.final_order(n))
    assert np.max(np.abs(got - O.dft_oracle(x))) < 1e-12


def test_layout_validation():
    with pytest.raises(ValueError):
        D.layout(6, 3)
    with pytest.raises(ValueError):
        D.layout(4, 8)  # needs n_local >= 2G+1
    assert D.layout(27, 8) == (30, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_local, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, G = D.layout(n_local, world)
        x = random_state(n, np.random.default_rng(11))
        slab = torch.from_numpy(np.split(x, world)[rank].copy())
        # exchange A with a real collective on the complex slab viewed as reals
        a = torch.view_as_real(slab).reshape(-1).contiguous()
        out = torch.empty_like(a)
        dist.all_to_all_single(out, a)
        cur = torch.view_as_complex(out.reshape(-1, 2)).numpy().copy()
        top, body = D.plans(n_local, world, rank, "c64")
        from paper_2304_14969_b200 import fusion
        fusion.run_plan_numpy(top, cur)
        a = torch.view_as_real(torch.from_numpy(cur)).reshape(-1).contiguous()
        out = torch.empty_like(a)
        dist.all_to_all_single(out, a)
        cur = torch.view_as_complex(out.reshape(-1, 2)).numpy().copy()
        fusion.run_plan_numpy(body, cur)
        mine = torch.view_as_real(torch.from_numpy(cur)).contiguous()  # gloo has no complex dtypes
        gathered = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
        dist.gather(mine, gathered, dst=0)
        if rank == 0:
            full = np.concatenate([torch.view_as_complex(g).numpy() for g in gathered])
            got = O.permute_qubits(full, D.final_order(n))
            q.put(float(np.max(np.abs(got - O.dft_oracle(x)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sharded_qft(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        err = q.get(timeout=120)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert err < 1e-12


# ---------------------------------------------------------------------------
# "virtual ranks" on one GPU: every rank's slab lives on cuda:0,
# the all-to-alls are device block transposes, and the per-rank top-layer and
# body programs run through the real kernels (k_sweep / k_qft) on sk_wrap
# views.  Checks the device path of the sharded QFT without a multi-GPU box.
# ---------------------------------------------------------------------------
def _virtual_sharded_qft(x: np.ndarray, world: int, dtype: str) -> np.ndarray:
    import ctypes as C

    from paper_2304_14969_b200 import _lib
    from paper_2304_14969_b200.executor import Program

    n = int(x.size).bit_length() - 1
    n_local = n - (world.bit_length() - 1)
    real = torch.float32 if dtype == "c64" else torch.float64
    cplx = np.complex64 if dtype == "c64" else np.complex128
    slabs = [torch.view_as_real(torch.from_numpy(s.astype(cplx))).reshape(-1).to("cuda").contiguous()
             for s in np.split(x, world)]
    torch.cuda.synchronize()
    _lib.call("sk_set_stream", 0, torch.cuda.current_stream().cuda_stream)

    def exchange(cur):  # all_to_all_single: out[r] block s = in[s] block r
        blocks = [c.view(world, -1) for c in cur]
        return [torch.cat([blocks[s][r] for s in range(world)]).contiguous() for r in range(world)]

    def run(prog, buf):
        h = C.c_void_p()
        _lib.call("sk_wrap", n_local, _lib.DTYPES[dtype], 0, buf.data_ptr(), C.byref(h))
        try:
            Program(prog, 0).run_handle(h)
        finally:
            _lib._lib.sk_destroy(h)

    cur = exchange(slabs)
    for r in range(world):
        top, _ = D.plans(n_local, world, r, dtype)
        run(top, cur[r])
    cur = exchange(cur)
    for r in range(world):
        _, body = D.plans(n_local, world, r, dtype)
        run(body, cur[r])
    torch.cuda.synchronize()
    out = np.concatenate([torch.view_as_complex(c.view(-1, 2)).cpu().numpy() for c in cur]).astype(complex)
    return O.permute_qubits(out, D.final_order(n))


@pytest.mark.gpu
@pytest.mark.parametrize("world,n_local", [(2, 9), (4, 10), (8, 11)])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_virtual_ranks_sharded_qft_on_device(rng, world, n_local, dtype):
    n, _ = D.layout(n_local, world)
    x = random_state(n, rng)
    got = _virtual_sharded_qft(x, world, dtype)
    tol = 1e-12 if dtype == "c128" else 1e-5
    assert np.max(np.abs(got - O.dft_oracle(x))) < tol


@pytest.mark.gpu
def test_virtual_ranks_sharded_qft_large_closed_form():
    # QFT-24 over 8 virtual ranks (2^21 per slab), GHZ input: y_j = (1 + e^{-2 pi i j/N}) / sqrt(2N)
    n, world = 24, 8
    x = np.zeros(1 << n, complex)
    x[0] = x[-1] = 2 ** -0.5
    got = _virtual_sharded_qft(x, world, "c64")
    assert np.max(np.abs(got - O.qft_of_ghz(n, np.arange(1 << n)))) < 1e-5


def _pairwise_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        slabs = [rng.normal(size=64 * world) for _ in range(world)]
        buf = torch.from_numpy(slabs[rank].copy())
        staging = torch.empty(7, dtype=buf.dtype)  # deliberately not a divisor of the block size
        D.pairwise_exchange(dist, buf, staging, world, rank)
        want = D.exchange_blocks([s.copy() for s in slabs])[rank]
        q.put((rank, float(np.max(np.abs(buf.numpy() - want)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_pairwise_inplace_exchange(world):
    """The in-place chunked pairwise exchange (one slab + a staging buffer,
    what QFT-37 needs at 128 GiB per GPU) equals all_to_all_single."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pairwise_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        errs = [q.get(timeout=120) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert max(e for _, e in errs) == 0.0


@pytest.mark.parametrize("world,n_local", [(2, 6), (4, 8), (8, 9)])
def test_one_exchange_schedule_emulated(rng, world, n_local):
    """One-exchange sharded QFT (rank = low G qubits): phase-shifted body on
    every rank, one all-to-all, the G-layer tail; kernel-op emulation of
    every sweep (tests/test_kernel_lowering.emulate) equals the DFT."""
    from test_kernel_lowering import emulate
    n, G = D.layout(n_local, world)
    x = random_state(n, rng)
    body, tail = D.plans_one_exchange(n_local, world, "c128")
    slabs = [emulate(body, x[r::world].copy(), pshift=G, pconst=r) for r in range(world)]
    slabs = D.exchange_blocks(slabs)
    slabs = [emulate(tail, s_.copy()) for s_ in slabs]
    u = np.empty(1 << n, complex)
    u[D.one_x_label(n_local, G)] = np.concatenate(slabs)
    got = O.permute_qubits(u, D.final_order(n))
    assert np.max(np.abs(got - O.dft_oracle(x))) < 1e-12


def _virtual_one_exchange(x: np.ndarray, world: int, dtype: str) -> np.ndarray:
    """One-exchange schedule with every rank on cuda:0 (real kernels: the
    phase-shifted k_qft body, the generic tail sweep)."""
    import ctypes as C

    from paper_2304_14969_b200 import _lib
    from paper_2304_14969_b200.executor import Program

    n = int(x.size).bit_length() - 1
    G = world.bit_length() - 1
    n_local = n - G
    cplx = np.complex64 if dtype == "c64" else np.complex128
    slabs = [torch.view_as_real(torch.from_numpy(x[r::world].astype(cplx))).reshape(-1).to("cuda").contiguous()
             for r in range(world)]
    torch.cuda.synchronize()
    _lib.call("sk_set_stream", 0, torch.cuda.current_stream().cuda_stream)
    body_plan, tail_plan = D.plans_one_exchange(n_local, world, dtype)
    tail = Program(tail_plan, 0)

    def run(prog, buf):
        h = C.c_void_p()
        _lib.call("sk_wrap", n_local, _lib.DTYPES[dtype], 0, buf.data_ptr(), C.byref(h))
        try:
            prog.run_handle(h)
        finally:
            _lib._lib.sk_destroy(h)

    for r in range(world):
        body = Program(body_plan, 0)
        body.set_phase_index(G, r)
        run(body, slabs[r])
    blocks = [c.view(world, -1) for c in slabs]
    slabs = [torch.cat([blocks[s][r] for s in range(world)]).contiguous() for r in range(world)]
    for r in range(world):
        run(tail, slabs[r])
    torch.cuda.synchronize()
    u = np.empty(1 << n, complex)
    u[D.one_x_label(n_local, G)] = np.concatenate([torch.view_as_complex(c.view(-1, 2)).cpu().numpy() for c in slabs])
    return O.permute_qubits(u, D.final_order(n))


@pytest.mark.gpu
@pytest.mark.parametrize("world,n_local", [(2, 9), (4, 12), (8, 14)])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_virtual_ranks_one_exchange_on_device(rng, world, n_local, dtype):
    n, _ = D.layout(n_local, world)
    x = random_state(n, rng)
    got = _virtual_one_exchange(x, world, dtype)
    assert np.max(np.abs(got - O.dft_oracle(x))) < (1e-12 if dtype == "c128" else 1e-5)


@pytest.mark.gpu
def test_virtual_ranks_one_exchange_large_closed_form():
    n, world = 25, 8  # 2^22 per slab: three-sweep body with the phase shift
    x = np.zeros(1 << n, complex)
    x[0] = x[-1] = 2 ** -0.5
    got = _virtual_one_exchange(x, world, "c64")
    assert np.max(np.abs(got - O.qft_of_ghz(n, np.arange(1 << n)))) < 1e-5


# ---------------------------------------------------------------------------
# ShardedQFT.run itself (the class bench.py --gpus N runs) in a real
# world-size-2 process group: both ranks on cuda:0, gloo with the
# host-staged exchange (NCCL cannot put two ranks on one device).
# ---------------------------------------------------------------------------
def _sharded_run_worker(rank, world, port, n_local, dtype, schedule, q, overlap=True, exchange="host"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2304_14969_b200 import _lib
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        _lib.call("sk_set_stream", 0, stream.cuda_stream)
        n, G = D.layout(n_local, world)
        x = random_state(n, np.random.default_rng(99))
        sq = D.ShardedQFT(n_local, dtype, exchange=exchange, schedule=schedule, overlap=overlap, chunk_bytes=4096)
        slab = D.scatter_input(x, world, rank, schedule)
        cplx = torch.complex64 if dtype == "c64" else torch.complex128
        sq.state.copy_(torch.view_as_real(torch.from_numpy(slab).to(cplx)).reshape(-1))
        sq.run(None, stream)
        torch.cuda.synchronize()
        mine = sq.state.cpu().double().contiguous()
        gathered = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
        dist.gather(mine, gathered, dst=0)
        if rank == 0:
            slabs = [torch.view_as_complex(g.view(-1, 2)).numpy() for g in gathered]
            u = D.assemble_output(slabs, n_local, G, schedule)
            got = O.permute_qubits(u, D.final_order(n))
            q.put(float(np.max(np.abs(got - O.dft_oracle(x)))))
    except Exception as exc:  # surface the failure instead of a queue timeout
        q.put(repr(exc))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("schedule,overlap,exchange", [("one", True, "host"), ("one", False, "host"),
                                                      ("one", True, "host-pairwise"), ("one", False, "host-pairwise"),
                                                      ("two", False, "host")])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sharded_qft_run_on_device(world, dtype, schedule, overlap, exchange):
    """distributed.ShardedQFT.run in a real 2- / 4-process group, vs the DFT of
    the global vector: the one-exchange schedule with the exchange overlapped
    with the last body sweep (block-by-block launches + per-block async
    send/recv), without it, and the two-exchange schedule."""
    n_local = 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_run_worker,
                         args=(r, world, port, n_local, dtype, schedule, q, overlap, exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        err = q.get(timeout=300)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert not isinstance(err, str), err
    assert err < (1e-12 if dtype == "c128" else 1e-5)


# ---------------------------------------------------------------------------
# distributed.ShardedState: general circuits on a state sharded by global
# bits, global<->local swaps by pairwise exchange, rank-predicate controls and
# rank-constant diagonals — real 2- and 4-process groups on one device
# ---------------------------------------------------------------------------
def _sharded_state_worker(rank, world, port, n, dtype, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2304_14969_b200 import _lib
        from paper_2304_14969_b200.circuit import build_ghz, build_qft, build_random_circuit, gate_matrix
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        _lib.call("sk_set_stream", 0, stream.cuda_stream)
        if kind == "random":
            circ = build_random_circuit(n, 10, 4242)
        else:  # GHZ then QFT: global-target H, global controls, label swaps
            g1, g2 = build_ghz(n), build_qft(n)
            from paper_2304_14969_b200.circuit import Circuit
            circ = Circuit(n, tuple(g1.gates) + tuple(g2.gates))
        st = D.ShardedState(n, dtype, exchange="host", chunk_bytes=4096)
        st.run(circ)
        torch.cuda.synchronize()
        norm2 = st.norm2()
        p1 = st.probability(n - 1, 1)
        full = st.gather()
        if rank == 0:
            x = np.zeros(1 << n, complex)
            x[0] = 1.0
            want = O.dense_run(circ.gates, x, gate_matrix)
            q.put((float(np.max(np.abs(full - want))), norm2, abs(p1 - O.probability(want, n - 1, 1)),
                   st.exchanges))
    except Exception as exc:
        q.put(repr(exc))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,n", [(2, 10), (4, 11)])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("kind", ["random", "ghz_qft"])
def test_gloo_sharded_state_circuits(world, n, dtype, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_state_worker, args=(r, world, port, n, dtype, kind, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = q.get(timeout=300)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert not isinstance(res, str), res
    err, norm2, perr, exchanges = res
    tol = 1e-12 if dtype == "c128" else 1e-5
    assert err < tol, (err, exchanges)
    assert abs(norm2 - 1.0) < (1e-12 if dtype == "c128" else 1e-5)
    assert perr < tol
    assert exchanges > 0  # global qubits really were brought home


# ---------------------------------------------------------------------------
# Distributed largest shard: the native engine SPMD over a
# process group; shards wider than local_max_width are split over the ranks.
# The decisions must be the reference engine's (tests/golden/engine.npz and
# the 54q SDRP goldens) on every rank.
# ---------------------------------------------------------------------------
def _dist_engine_worker(rank, world, port, local_max, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2304_14969_b200 import _lib
        from paper_2304_14969_b200.circuit import build_random_circuit
        from paper_2304_14969_b200.engine import EngineConfig, HybridState, OptFlags
        from paper_2304_14969_b200.errors import MemoryBudgetError
        torch.cuda.set_device(0)
        _lib.call("sk_set_stream", 0, torch.cuda.current_stream().cuda_stream)
        eg = np.load(Path(__file__).resolve().parent / "golden" / "engine.npz")
        results = []
        keys = sorted({k.rsplit("/", 1)[0] for k in eg.files if k.startswith("eng/")})
        for key in keys:
            w, dep, seed, budget = (int(v) for v in eg[f"{key}/spec"])
            if w < local_max + 2 or not bool(eg[f"{key}/ok"]):
                continue
            fl = OptFlags(*[bool(b) for b in eg[f"{key}/flags"]])
            cfg = EngineConfig(sdrp=float(eg[f"{key}/p"]), mem_budget=budget, rng_seed=seed, optimizations=fl)
            sim = HybridState(w, cfg, local_max_width=local_max)
            sim.apply_circuit(build_random_circuit(w, dep, seed))
            sim.flush_all()
            ket = sim.full_ket().amps
            results.append((key, sim.eps_record, sim.peak_amplitudes, [sim.stats[s] for s in
                            ("label_swaps", "kernels", "eliminated_controls", "merges", "splits")],
                            float(np.max(np.abs(ket - eg[f"{key}/ket"]))), sim.distribution))
        # a 54-qubit SDRP run at the golden's p_min (circuit 2, budget 2^18)
        g54 = eg["minsdrp/54_7_2/spec"]
        w, dep, seed, budget = (int(v) for v in g54)
        p_min = float(eg["minsdrp/54_7_2/res"][1])
        sim = HybridState(w, EngineConfig(sdrp=p_min, mem_budget=budget, rng_seed=seed), local_max_width=local_max + 4)
        sim.apply_circuit(build_random_circuit(w, dep, seed))
        sim.flush_all()
        results.append(("54q", sim.eps_record, sim.peak_amplitudes, sim.stats["merges"], 0.0, sim.distribution))
        q.put((rank, results))
    except Exception as exc:
        import traceback
        q.put((rank, repr(exc) + traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,local_max", [(2, 6), (4, 7)])
def test_gloo_distributed_largest_shard_engine(golden, world, local_max):
    eg = golden("engine")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_engine_worker, args=(r, world, port, local_max, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        out = dict(q.get(timeout=600) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    ref = out[0]
    assert len(ref) >= 10
    assert sum(d["dist_shards"] for *_, d in ref) >= 5 and sum(d["exchanges"] for *_, d in ref) >= 5, \
        [d for *_, d in ref]  # shards really were split over the ranks and rank bits swapped in
    assert ref[-1][-1]["dist_shards"] > 0  # the 54-qubit run too
    for key, eps, peak, stats, kerr, _ in ref:
        if key == "54q":
            np.testing.assert_allclose(eps, eg["minsdrp/54_7_2/eps"], atol=1e-9)
            assert peak == int(eg["minsdrp/54_7_2/res"][3])
            continue
        np.testing.assert_allclose(eps, eg[f"{key}/eps"], atol=1e-9, err_msg=key)
        assert peak == int(eg[f"{key}/peak"]), key
        assert stats == [int(v) for v in eg[f"{key}/stats"]], key
        assert kerr < 1e-10, (key, kerr)
    for r in range(1, world):  # every rank took the same decisions
        for a, b in zip(ref, out[r]):
            assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2], (r, a[0])
