"""Data-parallel selection (paper Fig. 1, select_next_data_parallel): device
construction time vs the reference CPU Engine at d198 / pr1002 (pr2392 GPU only)."""
import sys, time, json, os
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
from paper_1101_2678_b200 import aco
from pyoracle import RefEngine, synth_coords
for n in (198, 1002, 2392):
    prob = aco.build_problem(aco.synthetic_instance(n))
    eng = aco.Engine(prob, aco.RunConfig(params=aco.Parameters(m=0, seed=1), selection=aco.SelectionStrategy(aco.Selection(2))))
    ks = []
    for i in range(3):
        r = eng.run_iteration(); ks.append(r.construct_kernel_ms)
    print(json.dumps({"n": n, "gpu_construct_kernel_ms": ks[-1], "update_ms": r.update_ms, "desc": eng.describe()}), flush=True)
    eng.close()
    if n <= 1002:
        xs, ys = synth_coords(n)
        ref = RefEngine(xs, ys, m=0, seed=1, selection=2, deposit=0, workers=0)
        t0 = time.time(); rr = ref.run_iteration()
        print(json.dumps({"n": n, "ref_construct_ms": rr["construct_ms"], "cores": ref.workers}), flush=True)
