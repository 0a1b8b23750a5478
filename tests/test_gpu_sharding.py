"""Config 5's multi-GPU path with real engines: two ranks (gloo control plane,
both on cuda:0 — the pod has one GPU) serve 7 independent requests i mod 2,
each rank through one grouped engine (Engine.sparse_forward_grouped) over its
requests; rank 0 gathers per-request checksums, which must equal the oracle's
per-request sparse_forward outputs (SIGE_MATH_EXACT: bit-exact, so the
float64 sums match exactly)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
N_REQ = 7
FIX = ["rect5", "blob5", "rect15", "multi15"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fixture(orc_or_sb, i):
    return orc_or_sb.make_edit_fixture(FIX[i % len(FIX)], 1, 3, 64, 64, 40 + i)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import paper_2211_02048_b200 as sb
    from paper_2211_02048_b200 import sharding

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = sb.Model("mini_unet_gn")
        cfg = sb.default_config(dilate_full=25)

        def handler(ids):
            fx = [_fixture(sb, i) for i in ids]
            orig = torch.cat([o for o, _ in fx]).cuda()
            edited = torch.cat([e for _, e in fx]).cuda()
            eng = sb.Engine(model, batch=len(ids), math=sb.MATH_EXACT)
            eng.precompute(orig)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = eng.sparse_forward_grouped(edited, config=cfg)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            host = out.cpu().numpy().astype(np.float64)
            return [(ms, float(host[k].sum())) for k in range(len(ids))]

        res = sharding.serve_grouped(N_REQ, handler, group=8)
        if rank == 0:
            q.put([(r.request, r.rank, r.ms, r.checksum) for r in res])
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def test_grouped_engines_world2(orc):
    from paper_2211_02048_b200 import sharding

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = [sharding.RequestResult(*r) for r in rows]
    sharding.check_cover(results, N_REQ, 2)
    om = orc.model("mini_unet_gn")
    import paper_2211_02048_b200 as sb

    cfg = sb.default_config(dilate_full=25)
    for r in results:
        o, e = _fixture(orc, r.request)
        want, _ = om.sparse_forward(om.precompute(o), e, orc.difference_mask(o, e), cfg)
        assert r.checksum == float(want[0].astype(np.float64).sum()), r.request
