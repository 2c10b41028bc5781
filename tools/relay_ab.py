"""A/B of the roulette relay (leftover ants built in segments by several
warps) against the plain one-warp-per-ant launch, on one GPU.

    python tools/relay_ab.py [n:m[:G] ...]

Each case runs in two subprocesses (ACO_RELAY=0 and the default), prints the
median construction-kernel ms of 5 iterations after 2 warm-ups, and checks
that both produce the same tours (G > 1: rank 0 of G in external-exchange
mode, i.e. one GPU's shard)."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, sys
sys.path.insert(0, %r)
from paper_1101_2678_b200 import aco
n, m, G = %d, %d, %d
prob = aco.build_problem(aco.synthetic_instance(n))
eng = aco.Engine(prob, aco.RunConfig(params=aco.Parameters(m=m, seed=1), world=G, rank=0,
                                     selection=aco.SelectionStrategy(aco.Selection.roulette_full)))
ks, h = [], hashlib.sha256()
for i in range(7):
    r = eng.run_iteration()
    t, l = eng.ants()
    h.update(t.tobytes())
    if i >= 2:
        ks.append(r.construct_kernel_ms)
print(json.dumps({"kernel_ms": sorted(ks)[len(ks) // 2], "tours": h.hexdigest()[:16],
                  "desc": eng.describe()}))
"""


def run(n, m, G, relay):
    env = dict(os.environ)
    if not relay:
        env["ACO_RELAY"] = "0"
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, n, m, G)], env=env,
                         capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def main():
    cases = sys.argv[1:] or ["2392:2392", "2392:19136:8", "1002:1002", "2392:2392:2", "2392:2392:4"]
    rows = []
    for c in cases:
        parts = [int(x) for x in c.split(":")]
        n, m, G = parts[0], parts[1], parts[2] if len(parts) > 2 else 1
        a, b = run(n, m, G, False), run(n, m, G, True)
        row = {"n": n, "m": m, "G": G, "plain_ms": a["kernel_ms"], "relay_ms": b["kernel_ms"],
               "same_tours": a["tours"] == b["tours"], "relay_desc": b["desc"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
    return rows


if __name__ == "__main__":
    main()
