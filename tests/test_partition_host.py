"""Host-side logic of the element-row partitioned 2-D path, on CPU.

* the row split and the storage layout (ghost row on each side of every
  partition) that ``sisdc_op2d_create_part`` mirrors;
* multi-process (gloo, world size 2 and 3): the NCCL unique-id bootstrap,
  the halo exchange in the issue order of part2d.cu (``halo_schedule``) over
  real point-to-point messages -- every ghost row must equal the periodic
  neighbour's boundary row of the global field -- and the allreduce of the
  per-rank partial dot products.
The device side (the same exchange through NCCL and the split CG) is checked
against the single-domain path in tests/test_gpu_partition.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_18526_b200.dgsem2d import (bootstrap_id, from_storage, halo_schedule, part_layout, rank_rows,
                                           to_storage)


def test_rank_rows_cover_every_row_once():
    for ney in (1, 5, 8, 13, 1024):
        for R in range(1, min(ney, 9) + 1):
            rows = []
            for q in range(R):
                rb, rc = rank_rows(ney, R, q)
                assert rc >= 1
                rows.extend(range(rb, rb + rc))
            assert rows == list(range(ney))
            sizes = [rank_rows(ney, R, q)[1] for q in range(R)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        rank_rows(4, 5, 0)


def test_storage_roundtrip_all_local():
    rng = np.random.default_rng(0)
    nc, ney, nex, p1 = 4, 7, 3, 4
    g = rng.standard_normal((nc, ney, nex, p1, p1))
    parts = part_layout(ney, nex, p1, nc, 3, range(3))
    n = parts[-1][2] + nc * (parts[-1][1] + 2) * nex * p1 * p1
    vec = to_storage(g, parts, np.zeros(n))
    assert np.array_equal(from_storage(vec, parts, g.shape), g)
    # ghost rows untouched by the scatter
    for rb, rc, off in parts:
        v = vec[off:off + nc * (rc + 2) * nex * p1 * p1].reshape(nc, rc + 2, nex, p1, p1)
        assert not v[:, 0].any() and not v[:, -1].any()


def test_halo_schedule_pairs_self():
    """One rank: both sends go to itself and are matched in order with the two
    receives (first owned row -> top ghost, last owned row -> bottom ghost),
    i.e. the periodic wrap of a single domain."""
    sch = halo_schedule(0, 1)
    sends = [r for k, p, r in sch if k == "send"]
    recvs = [r for k, p, r in sch if k == "recv"]
    assert list(zip(sends, recvs)) == [("first", "top_ghost"), ("last", "bottom_ghost")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global(nc, ney, nex, p1):
    return np.arange(nc * ney * nex * p1 * p1, dtype=np.float64).reshape(nc, ney, nex, p1, p1) * 0.5 + 1.0


def _worker(rank, world, port, nc, ney, nex, p1, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # NCCL unique id bootstrap (the bytes rank 0 made reach every rank)
        uid = bootstrap_id(rank, world, lambda: bytes(range(128)))
        ok_id = uid == bytes(range(128))
        g = _global(nc, ney, nex, p1)
        parts = part_layout(ney, nex, p1, nc, world, [rank])
        rb, rc, _ = parts[0]
        vec = to_storage(g, parts, np.zeros(nc * (rc + 2) * nex * p1 * p1))
        st = vec.reshape(nc, rc + 2, nex, p1, p1)
        rowof = {"first": 1, "last": rc, "top_ghost": rc + 1, "bottom_ghost": 0}
        for c in range(nc):
            reqs = []
            for kind, peer, row in halo_schedule(rank, world):
                t = torch.from_numpy(st[c, rowof[row]])
                reqs.append(dist.isend(t, peer) if kind == "send" else dist.irecv(t, peer))
            for r in reqs:
                r.wait()
        top = np.array_equal(st[:, rc + 1], g[:, (rb + rc) % ney])
        bot = np.array_equal(st[:, 0], g[:, (rb - 1) % ney])
        # allreduce of the per-rank partial dot products (the CG's one collective)
        part = torch.tensor([float((st[:, 1:-1] ** 2).sum()), float(st[:, 1:-1].sum()), 1.0], dtype=torch.float64)
        dist.all_reduce(part)
        tot_ok = abs(part[0].item() - float((g ** 2).sum())) <= 1e-12 * float((g ** 2).sum()) and part[2].item() == world
        q.put((rank, ok_id, top, bot, tot_ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,ney", [(2, 5), (3, 7), (2, 2)])
def test_halo_exchange_gloo(world, ney):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 2, ney, 3, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == list(range(world))
    for rank, ok_id, top, bot, tot in res:
        assert ok_id, rank
        assert top and bot, (rank, top, bot)
        assert tot, rank


def _status_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_18526_b200.dgsem2d import agree_on_status
        clean = agree_on_status(-1, 0)
        # rank 1 saw a non-finite rhs in (global) element 17 and two failed solves, rank 2 element 5
        mine = {0: (-1, 0), 1: (17, 2), 2: (5, 1)}[rank]
        q.put((rank, clean, agree_on_status(*mine)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_failure_flags_agree_over_ranks(world):
    """the NaN / no-convergence flags are reduced over the ranks (element index: min;
    failed solves: max), so every rank of a partitioned run raises the same error."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_status_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (17, 2) if world == 2 else (5, 2)
    for rank, clean, agreed in res:
        assert clean == (-1, 0), rank
        assert agreed == want, (rank, agreed)
