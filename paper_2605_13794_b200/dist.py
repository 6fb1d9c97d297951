"""Host-side multi-rank plumbing (one process per GPU): process group, NCCL unique-id broadcast,
index-parity shards and max-over-ranks timing.  No compute: the per-view path runs in libbgs.

Works with any torch.distributed backend ("nccl" on the GPU box, "gloo" in the CPU tests).
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def env_rank_world() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: str, device: torch.device | None = None) -> tuple[int, int]:
    if not dist.is_initialized():
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return dist.get_rank(), dist.get_world_size()


def broadcast_bytes(payload: bytes | None, nbytes: int, device: torch.device, src: int = 0) -> bytes:
    """Rank `src` sends `payload` (exactly nbytes), every rank returns it (the NCCL unique id)."""
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank() == src:
        assert payload is not None and len(payload) == nbytes
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())


def max_over_ranks(x: float, device: torch.device) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values, device: torch.device) -> np.ndarray:
    t = torch.tensor(np.asarray(values, dtype=np.float64), device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return t.cpu().numpy()


def shard_ids(n: int, rank: int, world: int) -> np.ndarray:
    """Index-parity shard G^(m) = {i : i mod M = m}, in local order;
    local j holds global id j*M + m (the id the kernels write into records)."""
    return np.arange(rank, n, world, dtype=np.int64)
