"""Long-run stability: construction time and fallback counts over 300
iterations at pr2392 (python tools/long_run.py)."""
import sys, json
sys.path.insert(0, '.')
from paper_1101_2678_b200 import aco
prob = aco.build_problem(aco.synthetic_instance(2392))
eng = aco.Engine(prob, aco.RunConfig(params=aco.Parameters(m=0, seed=1), selection=aco.SelectionStrategy(aco.Selection.roulette_full)))
for it in range(300):
    r = eng.run_iteration()
    if it % 25 == 0 or it == 299:
        print(json.dumps({"it": it, "kernel_ms": round(r.construct_kernel_ms, 3), "update_ms": round(r.update_ms, 3), "fallbacks": r.fallbacks, "tier2": r.certified_fp64, "best": r.best_length}), flush=True)
