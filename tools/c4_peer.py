"""C4 over N B200s of one box (one process per GPU, device groups exchanging
over NVLink): python -m torch.distributed.run --nproc-per-node N
--master-addr 127.0.0.1 tools/c4_peer.py [arrivals] [--one-gpu] [--check]

Every rank generates the same trace (reference generator, seed 0) and calls
PeerGroup.run; rank 0 prints the decisions/s (device time, max over ranks)
and, with --check, compares the result field by field with the single-GPU
sharded engine on the same trace.  --one-gpu puts every rank on cuda:0 (a
functional check of the IPC path on a one-GPU box: the ranks' kernels then
time-slice one device, so it is slow)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("arrivals", type=int, nargs="?", default=20000)
    ap.add_argument("--gpus", type=int, default=16384)
    ap.add_argument("--one-gpu", action="store_true")
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2512_16099_b200 import abi
    from paper_2512_16099_b200.engine import Engine, generate_batch
    from paper_2512_16099_b200.model import SimConfig, preset
    from paper_2512_16099_b200.peer import PeerGroup, torch_allgather

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = 0 if args.one_gpu else int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    sp = preset("normal25")
    sp.mean_interarrival_s = 25.0 / 2048
    sp.job_count = args.arrivals
    batch = generate_batch(sp, 0, 1)
    cfg = SimConfig(gpu_count=args.gpus)
    eng = Engine(local)
    group = PeerGroup(eng, world, rank, args.arrivals, torch_allgather())
    dist.barrier()
    t0 = time.perf_counter()
    res = group.run(batch, cfg, abi.OUT_JOBS | abi.OUT_TIMELINE)
    secs = time.perf_counter() - t0
    t = torch.tensor([secs], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        r = res[0]
        ev = int(r.summary["handler_events"])
        out = {"config": f"C4: {args.gpus} GPUs, {args.arrivals} arrivals over {world} device groups",
               "status": r.code, "seconds": float(t.item()), "handler_events": ev,
               "decisions_per_s": ev / float(t.item()), "makespan_s": r.workload_makespan_s,
               "migrations": int(r.summary["migration_count"])}
        if args.check:
            ref = eng.run_batch(batch, [cfg], abi.OUT_JOBS | abi.OUT_TIMELINE)[0]
            diffs = [f for f in r.summary.dtype.names
                     if np.asarray(r.summary[f]).tobytes() != np.asarray(ref.summary[f]).tobytes()]
            if r.per_job.tobytes() != ref.per_job.tobytes():
                diffs.append("per_job")
            if r.frag_timeline.tobytes() != ref.frag_timeline.tobytes():
                diffs.append("timeline")
            out["identical_to_one_gpu"] = not diffs
            out["diffs"] = diffs
        print(json.dumps(out), flush=True)
    group.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
