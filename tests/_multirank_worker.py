"""One rank of tests/test_gpu_multirank.py (launched by torch.distributed.run,
one process per GPU, NCCL).  Runs the engine's own sharded protocol —
ncclCommInitRank over world ranks, per-iteration exchange inside
libaco_gpu.so — and compares it on rank 0 with a single-GPU colony.

    python -m torch.distributed.run --nproc-per-node W tests/_multirank_worker.py \
        OUT.json DEPOSIT WIRE N ITERS
"""
import hashlib
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out_path, deposit, wire, n, iters = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3]),
                                         int(sys.argv[4]), int(sys.argv[5]))
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1101_2678_b200 import aco

    prob = aco.build_problem(aco.synthetic_instance(n))

    def cfg(**kw):
        return aco.RunConfig(params=aco.Parameters(m=0, seed=3),
                             selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                             deposit=aco.DepositStrategy(aco.Deposit(deposit)),
                             wire=aco.Wire(wire), device=local, **kw)

    obj = [aco.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    eng = aco.Engine(prob, cfg(rank=rank, world=world, nccl_id=obj[0]))
    single = aco.Engine(prob, cfg()) if rank == 0 else None  # same wire (fp32 is sharded-only)
    report = {"world": world, "deposit": deposit, "wire": wire, "iterations": []}
    for it in range(iters):
        rec = eng.run_iteration()
        tours, lens = eng.ants()
        gathered = [None] * world if rank == 0 else None
        dist.gather_object((eng.ant_begin, tours, lens), gathered, dst=0)
        tau = eng.pheromone()
        digests = [None] * world if rank == 0 else None
        dist.gather_object(hashlib.sha256(tau.tobytes()).hexdigest(), digests, dst=0)
        best_tour = eng.best_tour()
        if rank == 0:
            srec = single.run_iteration()
            st, sl = single.ants()
            gathered.sort(key=lambda x: x[0])
            mt = np.concatenate([g[1] for g in gathered])
            ml = np.concatenate([g[2] for g in gathered])
            stau = single.pheromone()
            rel = float(np.max(np.abs(tau - stau) / np.abs(stau)))
            report["iterations"].append({
                "tours_equal": bool(np.array_equal(mt, st)),
                "lengths_equal": bool(np.array_equal(ml, sl)),
                "best_equal": rec.best_length == srec.best_length,
                "mean_equal": rec.mean_length == srec.mean_length,
                "best_so_far_equal": eng.best_length() == single.best_length(),
                "best_tour_equal": bool(np.array_equal(best_tour, single.best_tour())),
                "tau_identical_across_ranks": len(set(digests)) == 1,
                "tau_bit_equal_single": bool(np.array_equal(tau, stau)),
                "tau_max_rel": rel,
                "exchange_ms": rec.exchange_ms,
            })
        dist.barrier()
    report["describe"] = eng.describe()  # e.g. "exchange=multimem" or its fixed64 fallback
    eng.close()
    if rank == 0:
        single.close()
        with open(out_path, "w") as f:
            json.dump(report, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
