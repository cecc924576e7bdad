"""Multi-GPU runtime: one process per GPU, torch.distributed as the plumbing.

The planner shards every BaB iteration's children round-robin over the ranks
(child k -> rank k % world) and exchanges the packed per-child reports once
per iteration with an allgather (bp_set_exchange in include/babplan_cuda.h).
Every rank then replays the identical host pick / split / merge / prune on
the same data, so the picks are bit-exact to the single-GPU order; each
child's sampler stream is keyed by its global index, so the whole run is
independent of the number of GPUs.

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

    def allgather(self, send: np.ndarray) -> np.ndarray:
        torch = self.torch
        t = torch.from_numpy(np.ascontiguousarray(send, dtype=np.uint8)).to(self.device)
        out = torch.empty(self.world * t.numel(), dtype=torch.uint8, device=self.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy()

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
    dev._exchange = ex  # keep the callback alive as long as the device
    return ex
