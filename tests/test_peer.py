"""Multi-GPU device groups, host side (paper_2512_16099_b200/peer.py): the
world-size-2 gloo handshake that wires the peer inboxes (blobs all-gathered
in rank order), the GPU-range partition every rank derives, and the C-ABI
surface.  The device protocol itself is checked by the emulation
(test_emu_cluster.py::test_device_groups) and on the B200
(tools/c4_shards.py, tools/c4_peer.py)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2512_16099_b200 import engine, peer


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, size, out_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2512_16099_b200 import peer as pr

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank + 1]) * size
    allb = pr.exchange_blobs(blob, world, pr.torch_allgather(), size)
    if rank == 0:
        np.save(out_path, np.frombuffer(allb, np.uint8))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_handshake_orders_blobs_by_rank(tmp_path):
    size = int(peer._bind().msg_peer_handle_size())
    assert size == 4 * 64  # inbox + rank 0's job rows, summary, timeline (cudaIpcMemHandle_t)
    out = str(tmp_path / "blobs.npy")
    mp.spawn(_worker, args=(2, _free_port(), size, out), nprocs=2, join=True)
    got = np.load(out)
    assert got.tobytes() == bytes([1]) * size + bytes([2]) * size


def test_handshake_rejects_short_blobs():
    import pytest

    with pytest.raises(RuntimeError):
        peer.exchange_blobs(b"x", 2, lambda b: [b], 1)


def test_shard_ranges_partition_the_cluster():
    for G, world, S in ((16384, 8, 16), (16384, 2, 16), (640, 3, 2), (520, 4, 1), (1000, 8, 16)):
        ranges = [peer.shard_range(G, r, world, S, s) for r in range(world) for s in range(S)]
        assert ranges[0][0] == 0 and ranges[-1][1] == G
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        sizes = [hi - lo for lo, hi in ranges]
        assert max(sizes) - min(sizes) <= 1


def test_peer_entry_points_exported():
    L = engine.lib()
    for n in ("msg_peer_open", "msg_peer_export", "msg_peer_connect", "msg_run_peer", "msg_peer_close",
              "msg_peer_handle_size"):
        assert hasattr(L, n)
