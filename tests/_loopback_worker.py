"""One process, G engine contexts on one GPU (one thread per rank), the
engine's own sharded protocol over the in-process loopback NCCL
(tests/loopnccl, loaded through ACO_NCCL_LIB), compared with a single-context
colony.  Writes a JSON report; used by tests/test_gpu_loopback_multirank.py.

    ACO_NCCL_LIB=.../libloopnccl.so python tests/_loopback_worker.py OUT G DEPOSIT WIRE N ITERS [SEL]
"""
import hashlib
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out, G, deposit, wire, n, iters = sys.argv[1], *(int(x) for x in sys.argv[2:7])
    sel = int(sys.argv[7]) if len(sys.argv) > 7 else 0
    from paper_1101_2678_b200 import aco

    prob = aco.build_problem(aco.synthetic_instance(n))

    def cfg(**kw):
        return aco.RunConfig(params=aco.Parameters(m=0, seed=5, nn=8),
                             selection=aco.SelectionStrategy(aco.Selection(sel)),
                             deposit=aco.DepositStrategy(aco.Deposit(deposit)),
                             wire=aco.Wire(wire), **kw)

    nccl_id = aco.nccl_unique_id()
    engines = [None] * G
    errors = []

    def create(r):
        try:
            engines[r] = aco.Engine(prob, cfg(rank=r, world=G, nccl_id=nccl_id))
        except Exception as e:  # noqa: BLE001
            errors.append(f"rank {r}: {e!r}")

    ts = [threading.Thread(target=create, args=(r,)) for r in range(G)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    if errors:
        raise SystemExit("; ".join(errors))
    single = aco.Engine(prob, cfg())
    report = {"world": G, "deposit": deposit, "wire": wire, "selection": sel,
              "describe": engines[0].describe(), "iterations": []}
    for it in range(iters):
        recs = [None] * G

        def step(r):
            try:
                recs[r] = engines[r].run_iteration()
            except Exception as e:  # noqa: BLE001
                errors.append(f"rank {r} iteration {it}: {e!r}")

        ts = [threading.Thread(target=step, args=(r,)) for r in range(G)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        if errors:
            raise SystemExit("; ".join(errors))
        srec = single.run_iteration()
        parts = sorted((e.ant_begin, *e.ants()) for e in engines)
        mt = np.concatenate([p[1] for p in parts])
        ml = np.concatenate([p[2] for p in parts])
        st, sl = single.ants()
        taus = [e.pheromone() for e in engines]
        stau = single.pheromone()
        rel = float(np.max(np.abs(taus[0] - stau) / np.abs(stau)))
        report["iterations"].append({
            "tours_equal": bool(np.array_equal(mt, st)),
            "lengths_equal": bool(np.array_equal(ml, sl)),
            "best_equal": all(r.best_length == srec.best_length for r in recs),
            "mean_equal": all(r.mean_length == srec.mean_length for r in recs),
            "best_so_far_equal": all(e.best_length() == single.best_length() for e in engines),
            "best_tour_equal": all(np.array_equal(e.best_tour(), single.best_tour()) for e in engines),
            "tau_identical_across_ranks": len({hashlib.sha256(t.tobytes()).hexdigest() for t in taus}) == 1,
            "choice_identical_across_ranks": len({hashlib.sha256(e.choice().tobytes()).hexdigest()
                                                  for e in engines}) == 1,
            "tau_bit_equal_single": bool(np.array_equal(taus[0], stau)),
            "tau_max_rel": rel,
        })
    for e in engines:
        e.close()
    single.close()
    with open(out, "w") as f:
        json.dump(report, f)


if __name__ == "__main__":
    main()
