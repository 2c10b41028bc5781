"""A/B of the accumulate arithmetic on one GPU (update_ms by CUDA events):
fp64 reds into tau (ACO_WIRE_FP64) vs exact int64 fixed-point sums
(ACO_WIRE_FIXED64) at pr2392 m = n and m = 8n.
    python tools/wire_ab.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1101_2678_b200 import aco  # noqa: E402

prob = aco.build_problem(aco.synthetic_instance(2392))
for m in (0, 8 * 2392):
    for wire in (aco.Wire.fp64, aco.Wire.fixed64):
        cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=1),
                            selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                            deposit=aco.DepositStrategy(aco.Deposit.accumulate), wire=wire)
        with aco.Engine(prob, cfg) as eng:
            recs = [eng.run_iteration() for _ in range(8)][3:]
            print(f"m={eng.m} wire={wire.name:8s} update_ms={statistics.median(r.update_ms for r in recs):.4f} "
                  f"construct_ms={statistics.median(r.construct_ms for r in recs):.4f}", flush=True)
