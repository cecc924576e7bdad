"""Multi-GPU runtime: one process per GPU, torch.distributed as the plumbing.

The planner shards every BaB iteration's children round-robin over the ranks
(child k -> rank k % world).  Every rank keeps the pool's heads
(id, bounds, volume, width, owner) and replays pick_out / prune identically, so
the picks are bit-exact to the single-GPU order; full records (box, best, top
samples) live on their owner.  Per iteration: the owner of each picked parent
splits it and ships the child records to their search ranks (all-to-all), then
the children's heads are all-gathered (bp_set_exchange / bp_set_alltoall in
include/babplan_cuda.h).  Each child's sampler stream is keyed by its global
index, so the whole run is independent of the number of GPUs.

With an NCCL process group the library runs the exchange itself (NcclLink:
its own communicator, device-direct child records); with gloo (the CPU and
same-GPU tests) the torch.distributed hooks (Exchange) carry it.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _capi


class Exchange:
    """ctypes callback: allgather of a host byte buffer over a process group."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.dist, self.torch, self.group = dist, torch, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        backend = dist.get_backend(group)
        self.device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        self.bytes_sent = 0
        self.calls = 0
        self.c_fn = _capi.EXCHANGE_FN(self._call)
        self.c_a2a = _capi.ALLTOALL_FN(self._a2a)

    def allgather(self, send: np.ndarray) -> np.ndarray:
        torch = self.torch
        t = torch.from_numpy(np.ascontiguousarray(send, dtype=np.uint8)).to(self.device)
        out = torch.empty(self.world * t.numel(), dtype=torch.uint8, device=self.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy()

    def alltoallv(self, send: np.ndarray, send_bytes, recv_bytes) -> np.ndarray:
        torch = self.torch
        t = torch.from_numpy(np.ascontiguousarray(send, dtype=np.uint8)).to(self.device)
        out = torch.empty(int(sum(recv_bytes)), dtype=torch.uint8, device=self.device)
        self.dist.all_to_all_single(out, t, [int(x) for x in recv_bytes], [int(x) for x in send_bytes], group=self.group)
        return out.cpu().numpy()

    def _a2a(self, user, send_ptr, send_bytes_ptr, recv_ptr, recv_bytes_ptr) -> int:
        try:
            sb = [send_bytes_ptr[i] for i in range(self.world)]
            rb = [recv_bytes_ptr[i] for i in range(self.world)]
            total = int(sum(sb))
            send = np.ctypeslib.as_array((C.c_ubyte * max(total, 1)).from_address(send_ptr))[:total]
            got = self.alltoallv(send, sb, rb)
            if got.nbytes:
                C.memmove(recv_ptr, got.ctypes.data, got.nbytes)
            self.bytes_sent += total
            self.calls += 1
            return 0
        except Exception:  # never raise through the C-ABI
            return 1

    def _call(self, user, send_ptr, nbytes, recv_ptr) -> int:
        try:
            send = np.ctypeslib.as_array((C.c_ubyte * nbytes).from_address(send_ptr))
            got = self.allgather(send)
            C.memmove(recv_ptr, got.ctypes.data, got.nbytes)
            self.bytes_sent += nbytes
            self.calls += 1
            return 0
        except Exception:  # never raise through the C-ABI
            return 1


def shard_of(child: int, world: int) -> int:
    """Rank that searches and bounds child k of an iteration."""
    return child % world


class NcclLink:
    """Device-direct exchange (bp_set_nccl): the library's own NCCL communicator over NVLink /
    NVSwitch.  Child records go from the splitting GPU's pack buffer to the searching GPU in one
    grouped send / receive per iteration, with no Python callback and no host staging; the
    heads and status words (64 B per child) are all-gathered through small device buffers.
    torch.distributed only carries the 128-byte communicator id from rank 0."""

    def __init__(self, dev, rank: int, world: int, uid: bytes):
        self.rank, self.world = rank, world
        _capi.check(dev.lib.bp_set_nccl(dev.h, rank, world, uid))
        self.dev = dev

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _capi.check(_capi.load().bp_nccl_unique_id(buf))
        return buf.raw

    def selftest(self, nbytes: int = 4096) -> bool:
        """All-gather and all-to-all-v of nbytes-sized segments across the ranks, checked."""
        ok = C.c_int(0)
        _capi.check(self.dev.lib.bp_nccl_selftest(self.dev.h, int(nbytes), C.byref(ok)))
        return ok.value == 1


def nccl_single(dev) -> NcclLink:
    """A one-rank device-direct link (tests: the NCCL path on one GPU)."""
    return NcclLink(dev, 0, 1, NcclLink.unique_id())


def attach(dev, group=None, direct: Optional[bool] = None):
    """Shard dev's planner over the default (or given) process group: device-direct NCCL
    (NcclLink) when the group's backend is NCCL (BP_EXCHANGE=host keeps the staged hooks),
    else the torch.distributed hooks (Exchange; gloo in the CPU tests)."""
    import os

    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    if direct is None:
        direct = dist.get_backend(group) == "nccl" and os.environ.get("BP_EXCHANGE", "nccl") != "host"
    if direct:
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        # rank 0's id (or an empty one when it cannot make one: every rank then takes the staged hooks)
        try:
            uid = NcclLink.unique_id() if rank == 0 else bytes(128)
        except _capi.BabplanError:
            uid = bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast(t, src=src, group=group)
        uid = bytes(t.cpu().tolist())
        if any(uid):
            link = NcclLink(dev, rank, world, uid)
            dev._exchange = link
            return link
    ex = Exchange(group)
    _capi.check(dev.lib.bp_set_exchange(dev.h, ex.rank, ex.world, ex.c_fn, None))
    _capi.check(dev.lib.bp_set_alltoall(dev.h, ex.c_a2a))
    dev._exchange = ex  # keep the callback alive as long as the device
    return ex
