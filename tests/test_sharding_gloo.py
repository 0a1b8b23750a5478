"""World-size-2 gloo test of the request-sharded multi-GPU path (CPU only):
ownership is round-robin, every request is served exactly once, results and
max-over-ranks timings reach rank 0 — the same code path bench.py and
sharding.serve use over NCCL on the B200 box."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_02048_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_requests, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def handler(i):
            # deterministic per-request work standing in for one sparse edit
            g = torch.Generator().manual_seed(1000 + i)
            x = torch.rand(64, generator=g)
            return float(rank + 1), float(x.sum())

        res = sharding.serve(n_requests, handler)
        worst = sharding.max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put(([(r.request, r.rank, r.ms, r.checksum) for r in res], worst))
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def test_requests_for_rank():
    assert sharding.requests_for_rank(10, 4, 1) == [1, 5, 9]
    assert sum(len(sharding.requests_for_rank(64, 8, r)) for r in range(8)) == 64
    with pytest.raises(ValueError):
        sharding.requests_for_rank(4, 2, 2)


def test_serve_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 9
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, worst = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results = [sharding.RequestResult(*r) for r in rows]
    sharding.check_cover(results, n, 2)
    for r in results:
        g = torch.Generator().manual_seed(1000 + r.request)
        assert r.checksum == pytest.approx(float(torch.rand(64, generator=g).sum()))
        assert r.ms == r.rank + 1
    assert worst == 2.0


def test_groups_for_rank():
    assert sharding.groups_for_rank(64, 8, 3, 16) == [[3, 11, 19, 27, 35, 43, 51, 59]]
    assert sharding.groups_for_rank(10, 1, 0, 4) == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9]]
    assert sum(len(g) for r in range(4) for g in sharding.groups_for_rank(64, 4, r, 5)) == 64


def _grouped_worker(rank, world, port, n_requests, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def handler(ids):
            return [(float(len(ids)), float(torch.rand(8, generator=torch.Generator().manual_seed(i)).sum()))
                    for i in ids]

        res = sharding.serve_grouped(n_requests, handler, group=3)
        if rank == 0:
            q.put([(r.request, r.rank, r.ms, r.checksum) for r in res])
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def test_serve_grouped_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 11
    procs = [ctx.Process(target=_grouped_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results = [sharding.RequestResult(*r) for r in rows]
    sharding.check_cover(results, n, 2)
    for r in results:
        assert r.checksum == pytest.approx(float(torch.rand(8, generator=torch.Generator().manual_seed(r.request)).sum()))
