"""Row-staging probe (libaco_probe.so aco_probe_stage): algorithmic GB/s of
one-warp CTAs pulling 9.7 KB rows (pr2392 size) per dependent step, by path."""
import ctypes as C
import json
import os
import sys

lib = C.CDLL(os.path.join(os.path.dirname(__file__), "..", "paper_1101_2678_b200", "libaco_probe.so"))
lib.aco_probe_stage.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]
names = {0: "tma+lds (wait each step)", 1: "tma double-buffered + lds", 2: "ldg.nc direct",
         3: "lds only (resident)", 4: "ldg.nc L1::no_allocate",
         5: "tma as 4 bulk copies + lds", 6: "ldg, 2 rows in flight (independent)"}
modes = [int(a) for a in sys.argv[1:]] or list(range(7))
out = []
for mode in modes:
    for w in ([1, 4, 8, 11] if mode == 1 else [1, 4, 8] if mode == 6 else [1, 4, 8, 12, 16, 17]):
        g, ms = C.c_double(), C.c_double()
        rc = lib.aco_probe_stage(0, mode, w, 2000, C.byref(g), C.byref(ms))
        rec = {"mode": names[mode], "warps_per_sm": w, "gbps": round(g.value, 1), "ms": round(ms.value, 3), "rc": rc}
        out.append(rec)
        print(json.dumps(rec), flush=True)
