"""Multi-GPU plumbing over torch.distributed (one process per GPU).

torch.distributed only carries the 128-byte NCCL id from rank 0 to the other
ranks; the data path (owner routing, NCCL send/recv of events, all-reduce of
the per-level counts) runs inside libltl4c (ltl4c_verify after ltl4c_state_comm).
"""
from __future__ import annotations

import os


def rank_slice(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of a global trace held by `rank` (rank r's
    events precede rank r+1's, which the exchange relies on for slice order)."""
    per = (n_total + world - 1) // world
    lo = min(n_total, rank * per)
    return lo, min(n_total, lo + per)


def broadcast_id(make_id, group=None) -> bytes:
    """Rank 0 calls make_id() (128 bytes); every rank returns the same bytes."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        raw = make_id()
        assert len(raw) == 128
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev))
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def join(state, group=None) -> None:
    """Join `state` to an NCCL communicator spanning the torch.distributed group."""
    import torch.distributed as dist
    import paper_1411_2239_b200 as ltl4c
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nid = broadcast_id(ltl4c.nccl_unique_id, group)
    state.comm(nid, world, rank)


def local_rank() -> int:
    return int(os.environ.get("LOCAL_RANK", "0"))
