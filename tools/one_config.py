"""Run a few iterations of one configuration (for ncu launch lists / captures).
    python tools/one_config.py N M SELECTION DEPOSIT ITERS [G]
G > 1: rank 0 of G in external-exchange mode (the shard's kernels, no NCCL)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1101_2678_b200 import aco  # noqa: E402

n, m, sel, dep, iters = (int(x) for x in sys.argv[1:6])
G = int(sys.argv[6]) if len(sys.argv) > 6 else 1
prob = aco.build_problem(aco.synthetic_instance(n))
eng = aco.Engine(prob, aco.RunConfig(params=aco.Parameters(m=m, seed=1),
                                     selection=aco.SelectionStrategy(aco.Selection(sel)),
                                     deposit=aco.DepositStrategy(aco.Deposit(dep)),
                                     world=G, rank=0))
for _ in range(iters):
    r = eng.run_iteration()
    print(f"construct_kernel_ms={r.construct_kernel_ms:.4f} update_ms={r.update_ms:.4f}",
          eng.describe(), flush=True)
