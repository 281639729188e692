"""Multi-process plumbing for the generator-row-sharded engine (one process per GPU).

torch.distributed is the control plane only: rendezvous (env:// from torchrun), the hand-over
of the 128-byte ncclUniqueId that libqsr's own NCCL communicator is built from, timing as the
max over ranks, and assembling per-rank results on the host. Every byte of the data path
(pivot blocks, partial products, flags, records) moves inside libqsr over NCCL
(csrc/exchange.cu), never through these helpers.
"""
from __future__ import annotations

import os
from typing import Optional, Sequence, Tuple

import numpy as np


def init_from_env(backend: str = "nccl"):
    """(world, rank, local_rank, dist-or-None) from torchrun's environment."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return 1, 0, 0, None
    import torch
    import torch.distributed as dist
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return world, rank, local, dist


def _device_for(dist):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def share_bytes(dist, payload: Optional[bytes], src: int = 0) -> bytes:
    """Broadcast a small byte string from rank `src` to every rank."""
    if dist is None:
        return payload
    obj = [payload]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def share_nccl_id(dist, rank: int) -> bytes:
    """Rank 0 creates the ncclUniqueId (through libqsr's NCCL); every rank receives it."""
    from paper_2603_14641_b200 import quasar as q  # (absolute: bench.py loads this file by path)
    uid = q.nccl_unique_id() if rank == 0 else None
    return share_bytes(dist, uid)


def max_over_ranks(dist, value: float) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def combine_shard_planes(dist, arrays: Sequence[np.ndarray]) -> None:
    """In place: every rank wrote only its own shard's words into zero-initialised full-size
    buffers (ShardedEngine.tableau_planes); a bitwise-OR all-reduce gives every rank the whole
    tableau."""
    if dist is None:
        return
    import torch
    dev = _device_for(dist)
    for a in arrays:
        t = torch.from_numpy(a.view(np.int64)).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.BOR)
        a.view(np.int64)[:] = t.cpu().numpy()


def shot_word_range(shots: int, world: int, rank: int) -> Tuple[int, int]:
    """Shot-word slice [w0, w0 + nw) of rank `rank` for many-shot sampling sharded by shot
    (frames are independent per shot-word; the Philox key (q<<24)|j is global, frames.hpp:63)."""
    kf = (shots + 63) // 64
    if not 1 <= world <= kf:
        raise ValueError("world must be in [1, ceil(shots/64)]")
    w0 = kf * rank // world
    return w0, kf * (rank + 1) // world - w0
