"""Per-GPU update time of the gather deposit at G > 1 on one GPU: G virtual
shards in external-exchange mode (the test harness's exchange done with
device copies), rank 0's device time for
  replicated: aco_gpu_update folding every row over all m ants (k_rows_gather_warp
              + k_rows<DELTA>), after an all-gather of the whole succ/pred tables;
  row-sharded: aco_gpu_fold (rank 0's n/G rows) + aco_gpu_update (apply the
              all-gathered delta rows to every row),
plus the bytes each GPU would move over NVLink for either exchange.

    python tools/gather_rowshard.py [n m G ...]   (default: config 4 at G = 2/4/8)"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch

    from paper_1101_2678_b200 import aco
    from test_gpu_sharded import DevArray

    args = [int(x) for x in sys.argv[1:]] or [2392, 19136, 2, 2392, 19136, 4, 2392, 19136, 8,
                                              2392, 2392, 8]
    for n, m, G in zip(args[0::3], args[1::3], args[2::3]):
        prob = aco.build_problem(aco.synthetic_instance(n))

        def cfg(rank):
            return aco.RunConfig(params=aco.Parameters(m=m, seed=1),
                                 selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                                 deposit=aco.DepositStrategy(aco.Deposit.scatter_gather),
                                 world=G, rank=rank)

        shards = [aco.Engine(prob, cfg(r)) for r in range(G)]
        bufs = [e.exchange_buffers() for e in shards]
        S, P64 = bufs[0]["S"], bufs[0]["P64"]
        B = -(-n // G)
        sp = torch.cuda.ExternalStream(shards[0].stream_handle(), device="cuda")
        res = {"replicated": [], "row_sharded": []}
        for it in range(6):
            mode = "row_sharded" if it % 2 else "replicated"
            for e in shards:
                e.construct()
            torch.cuda.synchronize()
            for name in ("succ", "pred"):
                views = [torch.as_tensor(DevArray(b[name], (G, n, S), "<i4"), device="cuda") for b in bufs]
                for g in range(G):
                    for q in range(G):
                        if q != g:
                            views[q][g].copy_(views[g][g])
            views = [torch.as_tensor(DevArray(b["inv"], (G * S,), "<f8"), device="cuda") for b in bufs]
            for g in range(G):
                for q in range(G):
                    if q != g:
                        views[q][g * S:(g + 1) * S].copy_(views[g][g * S:(g + 1) * S])
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if mode == "row_sharded":
                with torch.cuda.stream(sp):
                    a.record(sp)
                shards[0].fold()
                with torch.cuda.stream(sp):
                    b.record(sp)
                b.synchronize()
                fold_ms = a.elapsed_time(b)
                for e in shards[1:]:
                    e.fold()
                deltas = [torch.as_tensor(DevArray(x["delta"], (G * B, P64), "<f8"), device="cuda")
                          for x in bufs]
                for g in range(G):
                    for q in range(G):
                        if q != g:
                            deltas[q][g * B:(g + 1) * B].copy_(deltas[g][g * B:(g + 1) * B])
                torch.cuda.synchronize()
            else:
                fold_ms = 0.0
            c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(sp):
                c.record(sp)
            shards[0].update()
            with torch.cuda.stream(sp):
                d.record(sp)
            d.synchronize()
            for e in shards[1:]:
                e.update()
            res[mode].append({"fold_ms": fold_ms, "update_ms": c.elapsed_time(d)})
            taus = [e.pheromone() for e in shards[:2]]
            assert np.array_equal(taus[0], taus[1])
        S_ = -(-m // G)
        out = {"n": n, "m": m, "G": G, "ants_per_gpu": S_}
        for k, v in res.items():
            v = v[1:]  # first of each is warm-up
            out[k + "_ms"] = round(statistics.median(x["fold_ms"] + x["update_ms"] for x in v), 4)
        out["replicated_exchange_MB"] = round((G - 1) * (2 * n * S_ * 4 + S_ * 8) / 1e6, 1)
        out["row_sharded_exchange_MB"] = round(((G - 1) * 2 * B * S_ * 4 + (G - 1) * S_ * 8 +
                                                (G - 1) * B * P64 * 8) / 1e6, 1)
        print(json.dumps(out), flush=True)
        for e in shards:
            e.close()


if __name__ == "__main__":
    main()
