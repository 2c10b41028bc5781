"""Device cost of the NCCL fp32 wire on the sharded atomic path: a one-rank
NCCL engine (world = 1 with an id runs the sharded protocol) for a few
iterations; run under an ncu launch list to read k_delta_pack and
k_rows<3> (MODE_DELTA32) per launch.
    python tools/pack_cost.py N SELECTION ITERS"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1101_2678_b200 import aco  # noqa: E402

n, sel, iters = (int(x) for x in sys.argv[1:4])
prob = aco.build_problem(aco.synthetic_instance(n))
cfg = aco.RunConfig(params=aco.Parameters(m=min(n, 1250), seed=1),
                    selection=aco.SelectionStrategy(aco.Selection(sel)),
                    deposit=aco.DepositStrategy(aco.Deposit.accumulate),
                    nccl_id=aco.nccl_unique_id())
with aco.Engine(prob, cfg) as eng:
    for _ in range(iters):
        r = eng.run_iteration()
        print(f"update_ms={r.update_ms:.4f} exchange_ms={r.exchange_ms:.4f}", flush=True)
