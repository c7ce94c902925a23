"""Multi-GPU plumbing for the row-sharded RBRP: one process per GPU,
torch.distributed for rendezvous only (the library's own NCCL communicator carries
the data-path collectives over NVLink / NVSwitch).

  partition_rows(n, world, rank)  contiguous, chunk-aligned row range of a rank
  unique_id(group)                NCCL unique id created on rank 0, broadcast to all
  Comm(device, group)             librbrp communicator (rbrp_comm_init / destroy)
  max_over_ranks(x, group)        max of a float over ranks (timing)
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import torch
import torch.distributed as dist

from . import rbrp as _rb

CHUNK = _rb.CHUNK


def partition_rows(n: int, world: int, rank: int, chunk: int = CHUNK) -> Tuple[int, int]:
    """(row_offset, n_local) of `rank`: the n rows cut into `world` contiguous ranges
    whose boundaries are multiples of `chunk` (the sampling chunk, so that chunk
    totals are owned by exactly one rank), as even as whole chunks allow."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    nch = (n + chunk - 1) // chunk
    lo = (nch * rank) // world
    hi = (nch * (rank + 1)) // world
    r0 = min(n, lo * chunk)
    r1 = min(n, hi * chunk)
    return r0, r1 - r0


def unique_id(group=None) -> bytes:
    """128-byte NCCL unique id: made on rank 0 (rbrp_comm_unique_id), broadcast with
    torch.distributed (gloo or nccl backend)."""
    obj = [None]
    if dist.get_rank(group) == 0:
        buf = ctypes.create_string_buffer(128)
        rc = _rb.lib().rbrp_comm_unique_id(buf)
        if rc:
            raise _rb.RBRPError(rc, "rbrp_comm_unique_id")
        obj[0] = bytes(buf.raw)
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
    return obj[0]


class Comm:
    """librbrp NCCL communicator for this process' GPU."""

    def __init__(self, device: torch.device, group=None, uid: Optional[bytes] = None):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = uid if uid is not None else unique_id(group)
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, 128)
        rc = _rb.lib().rbrp_comm_init(ctypes.byref(h), buf, self.world, self.rank,
                                      device.index if device.index is not None else 0)
        if rc:
            raise _rb.RBRPError(rc, "rbrp_comm_init")
        self.handle = h.value

    def close(self):
        if self.handle:
            _rb.lib().rbrp_comm_destroy(ctypes.c_void_p(self.handle))
            self.handle = None


def max_over_ranks(x: float, group=None, device=None) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def id_distributed(X_local: torch.Tensor, n_global: int, row_offset: int, comm: Comm, **kw):
    """rbrp_id on this rank's rows with the NCCL communicator: every rank gets the same S;
    W is this rank's rows."""
    return _rb.id(X_local, n_global=n_global, row_offset=row_offset, comm=comm.handle, **kw)
