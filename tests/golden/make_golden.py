"""Regenerates tests/golden/golden.json from the REFERENCE ITSELF.

Runs the reference's own headers, compiled unmodified into
oracle/_ref/libaco_ref.so (oracle/ref_harness.cpp, oracle/Makefile), on the
survey's synthetic instances and on proj/data/att48, and
records the values the oracle and the GPU engine are checked against.  Needs
/root/reference (build container only); the JSON it writes is committed and
is all the GPU box needs.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Reference, RefEngine, fnv1a64, synth_coords  # noqa: E402

DATA = "/root/reference/proj/data"


def trace(xs, ys, ewt, selection, deposit, iters, m=0, nn=30, random_start=False):
    e = RefEngine(xs, ys, ewt=ewt, m=m, nn=nn, seed=1, selection=selection, deposit=deposit,
                  workers=4, random_start=random_start)
    best, mean, tour_h = [], [], []
    for _ in range(iters):
        r = e.run_iteration()
        best.append(r["best_length"])
        mean.append(repr(float(r["mean_length"])))
        t, _ = e.tours()
        tour_h.append(fnv1a64(t))
    bl, bt = e.best()
    return {"selection": selection, "deposit": deposit, "iters": iters, "m": e.m, "nn": nn,
            "random_start": random_start, "best": best, "mean": mean, "tours_fnv": tour_h,
            "tau_fnv": fnv1a64(e.pheromone()), "choice_fnv": fnv1a64(e.choice()),
            "best_so_far": bl, "best_tour": bt.tolist()}


def main():
    R = Reference.get()
    out = {"_generated_by": "tests/golden/make_golden.py from oracle/_ref (reference headers)",
           "fnv": "FNV-1a-64 over the raw little-endian bytes of the C-contiguous array"}
    # Random123 Philox4x32-10 known-answer vectors + the survey's uniform_at check
    kats = [([0, 0, 0, 0], 0),
            ([0xFFFFFFFF] * 4, 0xFFFFFFFFFFFFFFFF),
            ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], 0xA4093822 | (0x299F31D0 << 32))]
    out["philox_kat"] = [{"ctr": c, "key": k, "out": R.philox(c, k).tolist()} for c, k in kats]
    rng = np.random.default_rng(7)
    samples = []
    for _ in range(64):
        s, it, ant, st, dr = (int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32)),
                              int(rng.integers(0, 2**32)), int(rng.integers(0, 2**32)),
                              int(rng.integers(0, 2**32)))
        samples.append([s, it, ant, st, dr, repr(float(R.uniform_at(s, it, ant, st, dr)))])
    samples.append([1, 0, 0, 1, 0, repr(float(R.uniform_at(1, 0, 0, 1, 0)))])
    out["uniform_at"] = samples

    # att48 (proj/data): coords through the reference parser, opt tour length
    with open(os.path.join(DATA, "att48.tsp")) as f:
        axs, ays, aewt = R.parse_instance(f.read())
    with open(os.path.join(DATA, "att48.opt.tour")) as f:
        opt = R.parse_tour(f.read())
    ad = R.build_problem(axs, ays, aewt)
    out["att48"] = {"xs": axs.tolist(), "ys": ays.tolist(), "ewt": aewt,
                    "opt_tour": opt.tolist(),
                    "opt_len": R.tour_length(ad, np.append(opt, opt[0])),
                    "dist_fnv": fnv1a64(ad), "tau0": repr(float(R.tau0(ad, 48))),
                    "trace_roulette_accumulate": trace(axs, ays, aewt, 0, 0, 10)}

    # synth198: the survey's golden configuration, every selection x deposit
    xs, ys = synth_coords(198)
    d = R.build_problem(xs, ys)
    out["synth198"] = {"coords_first_last": [xs[0], ys[0], xs[-1], ys[-1]],
                       "dist_fnv": fnv1a64(d), "max_d": int(d.max()),
                       "tau0": repr(float(R.tau0(d, 198))),
                       "nn30_fnv": fnv1a64(R.nn_lists(d, 30)),
                       "traces": [trace(xs, ys, 0, 0, 0, 10), trace(xs, ys, 0, 0, 1, 10),
                                  trace(xs, ys, 0, 1, 0, 10), trace(xs, ys, 0, 1, 3, 10),
                                  trace(xs, ys, 0, 2, 0, 3), trace(xs, ys, 0, 0, 1, 3, m=450),
                                  trace(xs, ys, 0, 0, 0, 3, random_start=True)]}
    # larger sizes: iteration-0 construction of a bounded ant subset + tables
    for n, ants in ((1002, 64), (2392, 16)):
        xs, ys = synth_coords(n)
        d = R.build_problem(xs, ys)
        tau0 = R.tau0(d, n)
        ch = R.choice(d, np.full((n, n), tau0))
        t, l = R.construct(d, ch, 1, 0, 0, ants)
        nnl = R.nn_lists(d, 30)
        tn, ln = R.construct(d, ch, 1, 0, 0, ants, selection=1, nn_lists=nnl)
        out[f"synth{n}"] = {"dist_fnv": fnv1a64(d), "max_d": int(d.max()), "tau0": repr(float(tau0)),
                            "choice0_fnv": fnv1a64(ch), "nn30_fnv": fnv1a64(nnl),
                            "ants": ants, "roulette_tours_fnv": fnv1a64(t),
                            "roulette_lengths": l.tolist(), "nn_tours_fnv": fnv1a64(tn),
                            "nn_lengths": ln.tolist()}
    # the reference's own RunReport JSON / bench CSV (report.hpp) for synth198
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "_ref/ref_report"], check=True)
    xs, ys = synth_coords(198)
    coords = f"{len(xs)}\n" + "".join(f"{x:.1f} {y:.1f}\n" for x, y in zip(xs, ys))
    for dep in (1, 3):
        subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_report"),
                        os.path.join(here, f"report_synth198_dep{dep}"), str(dep), "6"],
                       input=coords.encode(), check=True)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
