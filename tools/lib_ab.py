"""A/B of library builds (ACO_GPU_LIB_VARIANT) on the construction kernel:
median construct_kernel_ms / update_ms over 5 iterations after 2 warm-ups and
a hash of the tours (identical tours expected across builds).

    python tools/lib_ab.py CASES [variant.so ...]
    CASES = comma-separated n:m:sel[:G] (sel 0 roulette, 1 nn), e.g. 10000:0:1:8"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys, json, statistics, hashlib
sys.path.insert(0, %r)
from paper_1101_2678_b200 import aco
n, m, sel, G = %d, %d, %d, %d
prob = aco.build_problem(aco.synthetic_instance(n))
cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=1),
                    selection=aco.SelectionStrategy(aco.Selection(sel)), world=G, rank=0)
h = hashlib.sha256()
with aco.Engine(prob, cfg) as e:
    kw = {}
    if os.environ.get("LIB_AB_PINNED") == "1":  # tours streamed into pinned host memory
        import torch
        mloc = e.ant_end - e.ant_begin
        kw = dict(tours_out=torch.empty((mloc, n + 1), dtype=torch.int32, pin_memory=True).numpy(),
                  lengths_out=torch.empty(mloc, dtype=torch.int64, pin_memory=True).numpy())
    recs = []
    for i in range(7):
        recs.append(e.run_iteration(**kw))
        h.update(e.ants()[0].tobytes())
    recs = recs[2:]
    print(json.dumps({"kernel_ms": round(statistics.median(r.construct_kernel_ms for r in recs), 4),
                      "construct_ms": round(statistics.median(r.construct_ms for r in recs), 4),
                      "update_ms": round(statistics.median(r.update_ms for r in recs), 4),
                      "tours": h.hexdigest()[:12]}))
"""
cases = [tuple(int(x) for x in c.split(":")) for c in sys.argv[1].split(",")]
for c in cases:
    n, m, sel = c[:3]
    G = c[3] if len(c) > 3 else 1
    for lib in [""] + sys.argv[2:]:
        env = dict(os.environ)
        if lib:
            env["ACO_GPU_LIB_VARIANT"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, n, m, sel, G)], env=env,
                           capture_output=True, text=True)
        print(f"n={n} m={m} sel={sel} G={G} {os.path.basename(lib) or 'default'}",
              r.stdout.strip() or r.stderr[-1500:], flush=True)
