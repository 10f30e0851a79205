"""N>1 path on CPU: world-size-2 gloo ranks shard a trace ensemble by seed
(weak scaling, no data-path collective) and gather the per-trace summaries
on rank 0; the gathered result equals a single-process run of all seeds.
The per-rank compute here is the oracle's C port (CPU box, no GPU); on the
GPU box the same driver calls the CUDA engine (bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import refbind as rb

pytestmark = pytest.mark.skipif(not rb.port_available(), reason="oracle port not built")

TRACES_PER_RANK = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _port_run(batch, cfg):
    s, _ = rb.port_run_batch_summaries(batch, [cfg])
    return s


def _worker(rank, world, port, out_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2512_16099_b200 import ensemble
    from paper_2512_16099_b200.model import SimConfig, preset

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = preset("normal25")
    spec.job_count = 60
    local = ensemble.run_shard(spec, SimConfig(gpu_count=8), rank, TRACES_PER_RANK, run_fn=_port_run)
    allsum = ensemble.gather_summaries(local, world)
    if rank == 0:
        np.save(out_path, allsum.view(np.uint8))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_process(tmp_path):
    from paper_2512_16099_b200 import abi, ensemble
    from paper_2512_16099_b200.model import SimConfig, preset

    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    gathered = np.load(out).view(abi.SUMMARY_DTYPE)
    spec = preset("normal25")
    spec.job_count = 60
    from paper_2512_16099_b200.engine import generate_batch

    whole = _port_run(generate_batch(spec, 0, 2 * TRACES_PER_RANK), SimConfig(gpu_count=8))
    assert len(gathered) == 2 * TRACES_PER_RANK
    assert gathered.tobytes() == whole.tobytes()
    assert ensemble.rank_seeds(1, TRACES_PER_RANK) == (TRACES_PER_RANK, TRACES_PER_RANK)


NAMED_TOTAL = 13  # uneven: 7 + 6 traces


def _named_worker(rank, world, port, out_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2512_16099_b200 import ensemble
    from paper_2512_16099_b200.model import SimConfig, preset

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = preset("normal25")
    spec.job_count = 60
    local = ensemble.run_named_shard(spec, SimConfig(gpu_count=8), rank, world, NAMED_TOTAL, run_fn=_port_run)
    assert len(local) == ensemble.shard_range(rank, world, NAMED_TOTAL)[1] - ensemble.shard_range(rank, world,
                                                                                                   NAMED_TOTAL)[0]
    allsum = ensemble.gather_summaries(local, world)
    if rank == 0:
        np.save(out_path, allsum.view(np.uint8))
    else:
        assert allsum is None
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_named_ensemble_split_matches_single_process(tmp_path):
    """bench.py's N>1 headline: the named ensemble (seeds 0..T-1) cut into
    contiguous ranges of unequal length, gathered in rank order on rank 0,
    equals the one-process run of the whole ensemble."""
    from paper_2512_16099_b200 import abi, ensemble
    from paper_2512_16099_b200.engine import generate_batch
    from paper_2512_16099_b200.model import SimConfig, preset

    out = str(tmp_path / "gathered.npy")
    mp.spawn(_named_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    gathered = np.load(out).view(abi.SUMMARY_DTYPE)
    spec = preset("normal25")
    spec.job_count = 60
    whole = _port_run(generate_batch(spec, 0, NAMED_TOTAL), SimConfig(gpu_count=8))
    assert gathered.tobytes() == whole.tobytes()
    assert [ensemble.shard_range(r, 3, 10) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
