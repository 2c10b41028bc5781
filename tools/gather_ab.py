"""A/B of the gather fold between library builds (ACO_GPU_LIB_VARIANT): median
update_ms of the scatter-gather deposit (k_rows_gather_warp + k_rows<DELTA>)
at pr2392 with m = n and m = 8n on one GPU, after `warm` iterations.
    python tools/gather_ab.py [variant.so ...]"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, statistics
sys.path.insert(0, %r)
from paper_1101_2678_b200 import aco
prob = aco.build_problem(aco.synthetic_instance(2392))
out = {}
for m, warm in ((0, 3), (0, 40), (8 * 2392, 3)):
    cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=1),
                        selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                        deposit=aco.DepositStrategy(aco.Deposit.scatter_gather))
    with aco.Engine(prob, cfg) as e:
        recs = [e.run_iteration() for _ in range(warm + 5)][warm:]
        out[f"m={e.m},it>={warm}"] = round(statistics.median(r.update_ms for r in recs), 4)
print(json.dumps(out))
"""
for lib in [""] + sys.argv[1:]:
    env = dict(os.environ)
    if lib:
        env["ACO_GPU_LIB_VARIANT"] = os.path.abspath(lib)
    r = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True)
    print(lib or "default", r.stdout.strip() or r.stderr[-2000:], flush=True)
