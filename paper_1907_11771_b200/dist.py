"""Process-group plumbing for multi-GPU runs (one process per GPU).

torch.distributed carries only host-side coordination: the NCCL unique id the
library's own communicators are built from, barriers around timed regions and
the max-over-ranks of measured times.  The data path (halo exchange, combine)
runs inside libgbs_b200.so over NCCL.  Backend-agnostic so the same helpers
are exercised with gloo on CPU (tests/test_multirank.py).
"""

from __future__ import annotations

import os
from typing import Optional

import torch
import torch.distributed as dist


def env():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device: Optional[torch.device] = None) -> None:
    if dist.is_initialized():
        return
    kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
    dist.init_process_group(backend, **kw)


def active() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def broadcast_bytes(payload: Optional[bytes], src: int = 0) -> bytes:
    """Rank `src`'s bytes on every rank (e.g. the 128-byte ncclUniqueId)."""
    if not active():
        return payload
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def barrier(sync_cuda: bool = True) -> None:
    if active():
        dist.barrier()
    if sync_cuda and torch.cuda.is_available():
        torch.cuda.synchronize()


def max_over_ranks(x: float, device: Optional[torch.device] = None) -> float:
    """Max of a per-rank scalar (e.g. device time) over all ranks."""
    if not active():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device: Optional[torch.device] = None) -> float:
    if not active():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_objects(obj):
    """Every rank's picklable `obj`, in rank order (a one-element list on one process)."""
    if not active():
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def merge_clocks(per_rank):
    """One clocks record for a multi-GPU timed region from every rank's sampler output:
    the lowest per-rank median SM clock (the slowest GPU sets the max-over-ranks time), the
    union of throttle reasons, and each rank's own record."""
    if len(per_rank) == 1:
        return per_rank[0]
    sm = [c.get("sm_mhz") for c in per_rank if c.get("sm_mhz") is not None]
    mx = [c.get("sm_max_mhz") for c in per_rank if c.get("sm_max_mhz") is not None]
    reasons = sorted({r for c in per_rank for r in c.get("reasons", [])})
    return {"sm_mhz": min(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": reasons, "samples": sum(int(c.get("samples", 0)) for c in per_rank),
            "per_rank": per_rank}
