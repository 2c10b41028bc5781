"""World-size-2 (gloo, CPU) check of the ant-sharded iteration: the
decomposition the engine runs over NCCL (tests/sharding_model.py)
reproduces the single-process colony — tours identical, gather-path tau
bit-identical, atomic-path tau within 1e-5, best/mean identical."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, m, iters, out_path, force_two_stage=False):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from sharding_model import (INF, key_shift, owner_of, shard_range, shard_size, stage2_ant,
                                stats_key, two_stage, unpack_key)
    from pyoracle import Oracle, synth_coords

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    O = Oracle.get()
    xs, ys = synth_coords(n)
    d = O.build_dist(xs, ys)
    S = shard_size(m, world)
    a0, a1 = shard_range(m, world, rank)
    tau_g = np.full((n, n), O.tau0(d, m))
    tau_a = tau_g.copy()
    best_so_far = None
    trace = []
    for it in range(iters):
        # construction of the local shard, global ant ids
        tg, lg, _ = O.construct(d, O.choice(d, tau_g), 1, it, a0, a1)
        ta, la, _ = O.construct(d, O.choice(d, tau_a), 1, it, a0, a1)
        # stats (k_shard_key / k_shard_ant): packed (length << shift | ant) MIN,
        # or the two-stage MIN of the length then of the candidate ant
        staged = force_two_stage or two_stage(m, n, int(d.max()))
        sh = 0 if staged else key_shift(m)
        key = stats_key(int(lg.min()), int(np.argmin(lg)), a0, sh) if len(lg) else INF
        kt = torch.tensor([key], dtype=torch.int64)
        dist.all_reduce(kt, op=dist.ReduceOp.MIN)
        if staged:
            gbest = int(kt.item())
            cand = stage2_ant(int(lg.min()), int(np.argmin(lg)), a0, gbest) if len(lg) else INF
            at = torch.tensor([cand], dtype=torch.int64)
            dist.all_reduce(at, op=dist.ReduceOp.MIN)
            gant = int(at.item())
        else:
            gbest, gant = unpack_key(int(kt.item()), sh)
        k = torch.tensor([gant], dtype=torch.int64)
        s = torch.tensor([int(lg.sum())], dtype=torch.int64)
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        assert owner_of(gant, m, world) in range(world)
        # the owner's tour, replicated by an all-reduce MAX (k_owner_tour)
        tb = torch.from_numpy(tg[gant - a0].copy() if a0 <= gant < a1
                              else np.zeros(n + 1, np.int32))
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        best_tour = tb.numpy().copy()
        # gather path: all-gather tours (shard-major, padded to S) then fold in order
        pad = np.full((S, n + 1), -1, np.int32)
        pad[: a1 - a0] = tg
        lpad = np.ones(S, np.int64)
        lpad[: a1 - a0] = lg
        gt = [torch.zeros((S, n + 1), dtype=torch.int32) for _ in range(world)]
        gl = [torch.zeros(S, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gt, torch.from_numpy(pad))
        dist.all_gather(gl, torch.from_numpy(lpad))
        tours = np.concatenate([x.numpy() for x in gt])[:m]
        lens = np.concatenate([x.numpy() for x in gl])[:m]
        tau_g = O.update(tau_g, tours, lens, 0.5, 1)
        # atomic path: local delta, all-reduce(sum), tau = tau*keep + delta
        delta = O.update(np.zeros((n, n)), ta, la, 0.5, 0) if len(la) else np.zeros((n, n))
        dt = torch.from_numpy(delta)
        dist.all_reduce(dt, op=dist.ReduceOp.SUM)
        tau_a = tau_a * 0.5 + dt.numpy()
        assert np.array_equal(best_tour, tours[gant])
        trace.append((gbest, int(k.item()), int(s.item()), tours))
    if rank == 0:
        np.savez(out_path, tau_g=tau_g, tau_a=tau_a,
                 best=np.array([t[0] for t in trace]), owner=np.array([t[1] for t in trace]),
                 sums=np.array([t[2] for t in trace]), tours=np.stack([t[3] for t in trace]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,staged", [(60, False), (75, False), (75, True)])  # 75: 38 + 37
def test_two_rank_sharded_iteration_equals_single_process(tmp_path, oracle, m, staged):
    n, iters, world = 60, 3, 2
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(world, _free_port(), n, m, iters, out, staged), nprocs=world,
             join=True)
    got = np.load(out)
    from pyoracle import synth_coords

    xs, ys = synth_coords(n)
    d = oracle.build_dist(xs, ys)
    tau_g = np.full((n, n), oracle.tau0(d, m))
    tau_a = tau_g.copy()
    for it in range(iters):
        t, l, _ = oracle.construct(d, oracle.choice(d, tau_g), 1, it, 0, m)
        assert np.array_equal(got["tours"][it], t)
        assert got["best"][it] == l.min()
        assert got["owner"][it] == int(np.argmin(l))
        assert got["sums"][it] == l.sum()
        tau_g = oracle.update(tau_g, t, l, 0.5, 1)
        ta, la, _ = oracle.construct(d, oracle.choice(d, tau_a), 1, it, 0, m)
        tau_a = oracle.update(tau_a, ta, la, 0.5, 0)
    assert np.array_equal(got["tau_g"], tau_g)  # deterministic path: bitwise
    rel = np.abs(got["tau_a"] - tau_a) / np.abs(tau_a)
    assert rel.max() <= 1e-5


def _tie_worker(rank, world, port, shift, rows, out_path):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from sharding_model import INF, stage2_ant, stats_key, unpack_key

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    got = []
    for lens in rows:  # this rank's local lengths, shard [rank*S, rank*S + len)
        lens = np.asarray(lens[rank], np.int64)
        a0 = rank * 4
        bl, bi = int(lens.min()), int(np.argmin(lens))
        kt = torch.tensor([stats_key(bl, bi, a0, shift)], dtype=torch.int64)
        dist.all_reduce(kt, op=dist.ReduceOp.MIN)
        if shift == 0:
            at = torch.tensor([stage2_ant(bl, bi, a0, int(kt.item()))], dtype=torch.int64)
            dist.all_reduce(at, op=dist.ReduceOp.MIN)
            got.append((int(kt.item()), int(at.item())))
        else:
            got.append(unpack_key(int(kt.item()), shift))
    if rank == 0:
        np.save(out_path, np.array(got, np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shift", [0, 3])
def test_iteration_best_tie_rule_across_ranks(tmp_path, shift):
    # ties across ranks resolve to the lowest GLOBAL ant (engine.hpp:117-129);
    # shift 0 = the two-stage protocol for lengths too long to pack
    big = (1 << 61) - 5 if shift == 0 else 1000
    rows = [([7, 5, 9, 5], [5, 6, 5, 8]),          # tie 5: rank 0 ant 1
            ([9, 9, 9, 9], [4, 9, 4, 9]),          # rank 1 ant 4
            ([big, big, big, big], [big, big, big, big])]  # all equal: ant 0
    out = str(tmp_path / "tie.npy")
    mp.spawn(_tie_worker, args=(2, _free_port(), shift, rows, out), nprocs=2, join=True)
    got = np.load(out).tolist()
    assert got == [[5, 1], [4, 4], [big, 0]]


def test_shard_ranges_cover_colony():
    sys_path = os.path.join(ROOT, "tests")
    import sys

    sys.path.insert(0, sys_path)
    from sharding_model import owner_of, shard_range

    for m in (1, 7, 2392, 19136):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                a, b = shard_range(m, world, r)
                covered.extend(range(a, b))
                for k in range(a, b):
                    assert owner_of(k, m, world) == r
            assert covered == list(range(m))
