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

The exchange goes over NCCL (NVLink 5 / NVSwitch) when the process group is
NCCL, or gloo for the CPU / same-GPU tests.
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


def attach(dev, group=None) -> Optional[Exchange]:
    """Shard dev's planner over the default (or given) process group."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    ex = Exchange(group)
    _capi.check(dev.lib.bp_set_exchange(dev.h, ex.rank, ex.world, ex.c_fn, None))
    _capi.check(dev.lib.bp_set_alltoall(dev.h, ex.c_a2a))
    dev._exchange = ex  # keep the callback alive as long as the device
    return ex
