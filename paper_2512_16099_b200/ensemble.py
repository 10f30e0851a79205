"""Trace-ensemble sharding across GPUs.

Ensembles (C2, C3, C5) are independent traces, so N GPUs simulate N disjoint
shards with no data-path collective; one gather brings the per-trace
summaries to rank 0 at the end.  Weak scaling: every rank owns
`traces_per_rank` consecutive seeds.

One process per GPU (torchrun); torch.distributed carries only the final
gather (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from . import abi


def rank_seeds(rank: int, traces_per_rank: int, seed_base: int = 0):
    """(first seed, count) of a rank's shard."""
    return seed_base + rank * traces_per_rank, traces_per_rank


def gather_summaries(local: np.ndarray, world: int, device: Optional[str] = None) -> Optional[np.ndarray]:
    """Concatenate every rank's SUMMARY_DTYPE array on rank 0 (rank order).
    Shards must have equal length (weak scaling).  Returns None off rank 0."""
    import torch
    import torch.distributed as dist

    if world == 1 or not dist.is_initialized():
        return local
    raw = np.ascontiguousarray(local).view(np.uint8)
    t = torch.from_numpy(raw.copy())
    if device is not None:
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    if dist.get_rank() != 0:
        return None
    return np.concatenate([o.cpu().numpy().view(abi.SUMMARY_DTYPE) for o in out])


def run_shard(spec, cfg, rank: int, traces_per_rank: int, run_fn: Optional[Callable] = None,
              seed_base: int = 0) -> np.ndarray:
    """Simulate this rank's shard; returns its per-trace summaries.

    run_fn(batch, cfg) -> SUMMARY_DTYPE array; defaults to the CUDA engine
    on the rank's current device."""
    from .engine import generate_batch

    seed0, n = rank_seeds(rank, traces_per_rank, seed_base)
    batch = generate_batch(spec, seed0, n)
    if run_fn is None:
        from .engine import default_engine

        res = default_engine().run_batch(batch, [cfg], 0)
        return np.array(res.summaries, abi.SUMMARY_DTYPE)
    return run_fn(batch, cfg)
