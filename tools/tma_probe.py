"""TMA row-copy issue cost (modes: with / without the proxy fence, copy only) and completion latency (one warp alone, L2-resident
rows): aco_probe_tma for one 10 KB row (pr2392's streamed row) as K = 1, 2, 4
bulk copies.  python tools/tma_probe.py"""
import ctypes as C
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "paper_1101_2678_b200", "libaco_probe.so"))
L.aco_probe_tma.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                            C.POINTER(C.c_double)]
res = {}
MODES = {0: "fence+expect_tx+copy", 1: "expect_tx+copy", 2: "copy only"}
for floats in (2508, 1056):
    for mode in (0, 1, 2):
        for K in (1, 2, 4):
            a, b = C.c_double(), C.c_double()
            rc = L.aco_probe_tma(0, floats, K, mode, 4000, C.byref(a), C.byref(b))
            key = f"row{floats * 4}B_{MODES[mode]}_K{K}"
            res[key] = {"rc": rc, "issue_cycles": round(a.value, 1), "complete_cycles": round(b.value, 1)}
            print(json.dumps({key: res[key]}), flush=True)
