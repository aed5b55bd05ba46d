"""torch.distributed plumbing for multi-GPU layouts (one process per GPU).

Only bootstrap and timing live here: the NCCL unique id created by rank 0 is
broadcast over the process group, each rank builds its sharded context
(fdl_create_sharded: its upper-triangle tiles, replicated O(n) state), and
timings are reduced as the max over ranks.  All per-iteration exchanges run
inside libfdl over NCCL (include/fdl.h).  Works with the "nccl" backend on GPUs
and with "gloo" on CPU (tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _device():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def broadcast_bytes(data: bytes | None, nbytes: int, src: int = 0) -> bytes:
    """Broadcast `nbytes` bytes from rank `src` (e.g. the 128-byte ncclUniqueId)."""
    t = torch.zeros(nbytes, dtype=torch.uint8, device=_device())
    if dist.get_rank() == src:
        assert data is not None and len(data) == nbytes
        t.copy_(torch.tensor(list(data), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (multi-GPU timings are reported as the max)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_in_rank_order(values) -> float:
    """Gather one float per rank and sum in rank order (deterministic)."""
    t = torch.tensor([float(values)], dtype=torch.float64, device=_device())
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    s = 0.0
    for x in out:
        s += float(x.item())
    return s


def sharded_layout(g, params, init_pos, edge_len=None):
    """Build this rank's context of a world-size layout (NCCL over NVLink)."""
    from . import fdl

    rank, world = dist.get_rank(), dist.get_world_size()
    nid = fdl.nccl_unique_id() if rank == 0 else None
    nid = broadcast_bytes(nid, 128, 0)
    return fdl.Layout.from_graph(g, params=params, init_pos=init_pos, nccl_id=nid, rank=rank, world=world,
                                 edge_len=edge_len)
