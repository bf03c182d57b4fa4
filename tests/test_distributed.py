"""Global-qubit sharded QFT (host logic, CPU): the per-rank plans plus the
all-to-all block exchange reproduce the oracle DFT; the exchange semantics
are checked against a real world-size-2/4 gloo all_to_all_single."""
from __future__ import annotations

import os
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
