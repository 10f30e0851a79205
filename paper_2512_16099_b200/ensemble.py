"""Trace-ensemble sharding across GPUs.

Ensembles (C2, C3, C5) are independent traces, so N GPUs simulate N disjoint
shards with no data-path collective; one gather brings the per-trace
summaries to rank 0 at the end.  Two ways to cut the work:

* named ensemble, split (strong scaling): the ensemble BASELINE.json names
  (e.g. C2's seeds 0..4095) cut into N contiguous trace ranges
  (`shard_range`), so the gathered result is exactly the one-GPU result;
* weak scaling: every rank owns `traces_per_rank` consecutive seeds
  (`rank_seeds`).

One process per GPU (torchrun); torch.distributed carries only the final
gather (NCCL on GPUs, gloo in the CPU tests).  The reference itself runs
independent traces in separate processes; results do not
depend on how traces are placed on devices (test_sim_engine.cpp:172-182).
"""
from __future__ import annotations

import os
from typing import Callable, Optional

import numpy as np

from . import abi


def rank_seeds(rank: int, traces_per_rank: int, seed_base: int = 0):
    """(first seed, count) of a rank's shard under weak scaling."""
    return seed_base + rank * traces_per_rank, traces_per_rank


def shard_range(rank: int, world: int, total: int):
    """[lo, hi) of a rank's contiguous share of `total` traces (the first
    total % world ranks get one more)."""
    q, r = divmod(total, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def local_device() -> int:
    """The CUDA device of this rank: torch's current device when CUDA is
    initialised, else LOCAL_RANK (torchrun), else 0."""
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return torch.cuda.current_device()
    except Exception:
        pass
    return int(os.environ.get("LOCAL_RANK", "0"))


def gather_summaries(local: np.ndarray, world: int, device: Optional[str] = None) -> Optional[np.ndarray]:
    """Concatenate every rank's SUMMARY_DTYPE array on rank 0 in rank order
    (shards may differ in length).  Returns None off rank 0."""
    out = gather_records(np.ascontiguousarray(local, abi.SUMMARY_DTYPE), world, device)
    return out


def gather_records(local: np.ndarray, world: int, device: Optional[str] = None) -> Optional[np.ndarray]:
    """Rank-ordered concatenation on rank 0 of a structured array whose
    length may differ by rank: one all-gather of the lengths, one of the
    records padded to the longest shard."""
    import torch
    import torch.distributed as dist

    if world == 1 or not dist.is_initialized():
        return local
    dtype = local.dtype
    raw = np.ascontiguousarray(local).view(np.uint8)
    n = torch.tensor([len(local)], dtype=torch.int64, device=device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    lens = [int(x.item()) for x in ns]
    cap = max(lens) * dtype.itemsize
    buf = np.zeros(max(cap, 1), np.uint8)
    buf[:raw.size] = raw
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    if dist.get_rank() != 0:
        return None
    parts = [o.cpu().numpy()[:k * dtype.itemsize].view(dtype) for o, k in zip(out, lens)]
    return np.concatenate(parts) if parts else np.zeros(0, dtype)


def run_shard(spec, cfg, rank: int, traces_per_rank: int, run_fn: Optional[Callable] = None,
              seed_base: int = 0, engine=None) -> np.ndarray:
    """Simulate this rank's weak-scaling shard; returns its per-trace
    summaries.

    run_fn(batch, cfg) -> SUMMARY_DTYPE array; defaults to the CUDA engine
    of this rank's device (`engine`, else default_engine(local_device()))."""
    from .engine import generate_batch

    seed0, n = rank_seeds(rank, traces_per_rank, seed_base)
    return _run(generate_batch(spec, seed0, n), cfg, run_fn, engine)


def run_named_shard(spec, cfg, rank: int, world: int, total: int, run_fn: Optional[Callable] = None,
                    seed_base: int = 0, engine=None) -> np.ndarray:
    """Simulate this rank's contiguous share of the named ensemble (seeds
    seed_base .. seed_base + total - 1); returns its per-trace summaries.
    Gathered in rank order they are the summaries of the whole ensemble."""
    from .engine import generate_batch

    lo, hi = shard_range(rank, world, total)
    return _run(generate_batch(spec, seed_base + lo, hi - lo), cfg, run_fn, engine)


def _run(batch, cfg, run_fn, engine):
    if run_fn is not None:
        return run_fn(batch, cfg)
    if engine is None:
        from .engine import default_engine

        engine = default_engine(local_device())
    res = engine.run_batch(batch, [cfg], 0)
    return np.array(res.summaries, abi.SUMMARY_DTYPE)
