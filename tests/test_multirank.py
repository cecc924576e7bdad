"""N>1 path on CPU: world_size-2 gloo process groups exercising the exchange
hook the sharded planner calls (paper_2412_09584_b200.parallel)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2412_09584_b200 import parallel


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = parallel.Exchange()
        # rank-ordered allgather through the ctypes callback the C library calls
        send = (np.arange(37, dtype=np.uint8) * (rank + 1)).astype(np.uint8)
        recv = np.zeros(37 * world, dtype=np.uint8)
        rc = ex.c_fn(None, send.ctypes.data, send.nbytes, recv.ctypes.data)
        want = np.concatenate([(np.arange(37, dtype=np.uint8) * (r + 1)).astype(np.uint8) for r in range(world)])
        ok1 = rc == 0 and np.array_equal(recv, want)
        # every child of an iteration lands on exactly one rank
        mine = [k for k in range(11) if parallel.shard_of(k, world) == rank]
        got = ex.allgather(np.array(mine + [255] * (6 - len(mine)), dtype=np.uint8))
        covered = sorted(int(x) for x in got if x != 255)
        ok2 = covered == list(range(11))
        # all-to-all-v through the ctypes callback: rank r sends (r+1)*10 + dst, dst+1 bytes to dst
        sb = np.array([dst + 1 for dst in range(world)], dtype=np.int64)
        send = np.concatenate([np.full(dst + 1, (rank + 1) * 10 + dst, dtype=np.uint8) for dst in range(world)])
        rb = np.array([rank + 1] * world, dtype=np.int64)
        recv = np.zeros(int(rb.sum()), dtype=np.uint8)
        rc = ex.c_a2a(None, send.ctypes.data, sb.ctypes.data_as(C.POINTER(C.c_int64)), recv.ctypes.data,
                      rb.ctypes.data_as(C.POINTER(C.c_int64)))
        want = np.concatenate([np.full(rank + 1, (src + 1) * 10 + rank, dtype=np.uint8) for src in range(world)])
        ok3 = rc == 0 and np.array_equal(recv, want)
        q.put((rank, bool(ok1), bool(ok2 and ok3)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_exchange_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=100) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    assert res == [(0, True, True), (1, True, True)]
