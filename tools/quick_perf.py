"""Quick device timing of the iteration at a given size (development tool)."""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def probe(bytes_, reps=20, iters=5):
    L = C.CDLL(os.path.join(ROOT, "paper_1101_2678_b200", "libaco_probe.so"))
    L.aco_probe_read_bw.argtypes = [C.c_int, C.c_size_t, C.c_int, C.c_int,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]
    g, ms = C.c_double(), C.c_double()
    rc = L.aco_probe_read_bw(0, bytes_, reps, iters, C.byref(g), C.byref(ms))
    return rc, g.value, ms.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2392)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--deposit", type=int, default=0)
    ap.add_argument("--selection", type=int, default=0)
    ap.add_argument("--stream", type=int, default=0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--probe", action="store_true")
    a = ap.parse_args()
    if a.probe:
        for mb in (16, 32, 48, 64, 96, 2048):
            print("read_bw", mb, "MB", probe(mb << 20, reps=20 if mb < 200 else 3))
    from paper_1101_2678_b200 import aco

    spec = aco.synthetic_instance(a.n)
    prob = aco.build_problem(spec)
    cfg = aco.RunConfig(params=aco.Parameters(m=a.m, seed=1),
                        selection=aco.SelectionStrategy(aco.Selection(a.selection)),
                        deposit=aco.DepositStrategy(aco.Deposit(a.deposit)),
                        stream=aco.WeightStream(a.stream))
    t0 = time.time()
    eng = aco.Engine(prob, cfg)
    print("create s", time.time() - t0, "stream", eng.weight_stream)
    for i in range(a.warmup + a.iters):
        r = eng.run_iteration()
        print(json.dumps({"it": r.iteration, "best": r.best_length, "construct_ms": round(r.construct_ms, 3),
                          "kernel_ms": round(r.construct_kernel_ms, 3), "update_ms": round(r.update_ms, 3),
                          "choice_ms": round(r.choice_ms, 3), "fallbacks": r.fallbacks}))
    eng.close()


if __name__ == "__main__":
    main()
