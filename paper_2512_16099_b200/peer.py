"""Multi-GPU device groups: one large trace (C4: 16384 simulated GPUs, 1M
arrivals) split over the B200s of one NVLink/NVSwitch domain, one process per
GPU (include/migsched_b200.h, msg_peer_*).

Each rank owns a contiguous range of the simulated cluster's GPUs; every
decision (next event, placement, plan_inter source, the departed GPU's class)
is an all-reduce of packed keys done by the kernels themselves through
peer-mapped inboxes — the host only wires the inboxes up once:

    group = PeerGroup(engine, world, rank, max_jobs, allgather)
    result = group.run(batch, cfg)      # BatchResult on rank 0, None elsewhere

`allgather(bytes) -> list[bytes]` exchanges one blob per rank in rank order;
`torch_allgather()` builds it from an initialised torch.distributed group
(gloo or NCCL: only the setup handshake goes through it).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional

from . import abi
from .engine import BatchResult, Engine, _check, _decode, lib
from .model import ConfigPack, SimConfig, TraceBatch

_bound = False


def _bind():
    global _bound
    L = lib()
    if not _bound:
        vp, i32, u32, u64 = C.c_void_p, C.c_int32, C.c_uint32, C.c_uint64
        for name, res, args in (
            ("msg_peer_handle_size", C.c_size_t, []),
            ("msg_peer_open", C.c_int, [vp, i32, i32, u64, C.POINTER(vp)]),
            ("msg_peer_export", C.c_int, [vp, vp]),
            ("msg_peer_connect", C.c_int, [vp, vp]),
            ("msg_run_peer", C.c_int, [vp, vp, vp, vp, u32, C.POINTER(vp)]),
            ("msg_peer_close", None, [vp]),
        ):
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _bound = True
    return L


def shard_range(gpu_count: int, rank: int, world: int, shards: int = 1, shard: int = 0):
    """GPU range [lo, hi) owned by CTA `shard` of rank `rank`'s cluster: the
    global shard rank * shards + shard of world * shards splits the cluster
    into contiguous, balanced ranges (cluster_core.cuh, setup)."""
    gs, ns = rank * shards + shard, world * shards
    return gpu_count * gs // ns, gpu_count * (gs + 1) // ns


def torch_allgather(group=None) -> Callable[[bytes], List[bytes]]:
    """All-gather of one bytes blob per rank over torch.distributed."""
    import torch.distributed as dist

    def gather(blob: bytes) -> List[bytes]:
        out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, blob, group=group)
        return [bytes(b) for b in out]

    return gather


def exchange_blobs(blob: bytes, world: int, allgather: Callable[[bytes], List[bytes]], size: int) -> bytes:
    """Every rank's blob, concatenated in rank order (validated)."""
    blobs = allgather(blob)
    if len(blobs) != world or any(len(b) != size for b in blobs):
        raise RuntimeError(f"peer handshake: expected {world} blobs of {size} bytes, got "
                           f"{[len(b) for b in blobs]}")
    return b"".join(blobs)


class PeerGroup:
    """This rank's member of a multi-GPU device group (msg_peer)."""

    def __init__(self, engine: Engine, world: int, rank: int, max_jobs: int,
                 allgather: Callable[[bytes], List[bytes]]):
        L = _bind()
        self.engine = engine
        self.world, self.rank = world, rank
        h = C.c_void_p()
        _check(L.msg_peer_open(engine._h, world, rank, max_jobs, C.byref(h)), engine)
        self._h = h
        size = int(L.msg_peer_handle_size())
        buf = (C.c_char * size)()
        _check(L.msg_peer_export(self._h, buf), engine)
        allb = exchange_blobs(bytes(buf), world, allgather, size)
        _check(L.msg_peer_connect(self._h, C.c_char_p(allb)), engine)

    def run(self, batch: TraceBatch, cfg: SimConfig, out_flags: int = abi.OUT_JOBS) -> Optional[BatchResult]:
        """migsched::run of the batch's single trace over all ranks; every
        rank must call it with the same inputs.  Result on rank 0."""
        pack = ConfigPack([cfg])
        r = C.c_void_p()
        _check(_bind().msg_run_peer(self.engine._h, self._h, C.addressof(batch._c), C.addressof(pack.c[0]),
                                    out_flags, C.byref(r)), self.engine)
        return _decode(r, out_flags) if r.value else None

    def close(self):
        if self._h:
            _bind().msg_peer_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
