"""Sharded planner on the GPU: two and three ranks (processes) on one B200 over
gloo -- replicated pool heads, child records shipped from their parent's owner
to their search rank (all-to-all), children's heads all-gathered -- must
reproduce the single-process plan exactly (children keyed by global index,
identical host decisions on every rank)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    from paper_2412_09584_b200 import workloads
    wl = workloads.c1()
    cfg = wl.planner_config()
    cfg["batch"] = 8
    cfg["termination"]["max_iterations"] = 5
    cfg["search"]["samples_per_iter"] = 128
    cfg["search"]["iterations"] = 4
    return wl, cfg


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_09584_b200 as bp
        from paper_2412_09584_b200 import parallel

        wl, cfg = _cfg()
        dev = bp.Device(0).load(wl.spec)
        ex = parallel.attach(dev)
        res = dev.plan(cfg)
        q.put((rank, res["objective"], res["action"].tolist(), res["trace"]["uf"], res["trace"]["min_lf"],
               res["trace"]["pool_size"], res["samples"], ex.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_ranks_reproduce_single_process_plan(world):
    import paper_2412_09584_b200 as bp

    wl, cfg = _cfg()
    single = bp.Device(0).load(wl.spec).plan(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=250) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, obj, act, uf, mlf, pool, samples, calls in res:
        assert calls == 1 + 3 * 5  # root head; per iteration a status word, one all-to-all and one allgather
        assert obj == single["objective"] and np.array_equal(act, single["action"])
        assert uf == single["trace"]["uf"] and mlf == single["trace"]["min_lf"]
        assert pool == single["trace"]["pool_size"] and samples == single["samples"]


def _fail_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_09584_b200 as bp
        from paper_2412_09584_b200 import objective as objmod
        from paper_2412_09584_b200 import parallel

        wl, cfg = _cfg()
        spec = wl.spec
        big = objmod.ObjectiveSpec(**{**spec.__dict__, "W": [spec.W[0] * 1e30] + list(spec.W[1:])})
        dev = bp.Device(0).load(big)
        parallel.attach(dev)
        try:
            dev.plan(cfg)
            q.put((rank, "no error"))
        except RuntimeError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_rank_local_failure_raises_on_every_rank():
    """A failure on one rank (the root search on rank 0 overflows) reaches every rank through the
    status word of the next collective: all ranks raise, none is left blocked in the exchange."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_fail_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=250) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert "root search failed" in res[0]
    assert "rank 0 failed" in res[1]
