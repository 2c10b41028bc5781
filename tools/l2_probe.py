"""L2 read-bandwidth sweep: ld.global.nc (may hit in L1 on repeats) vs
ld.global.cg (L2 only), over resident buffer sizes."""
import ctypes as C
import json
import os

lib = C.CDLL(os.path.join(os.path.dirname(__file__), "..", "paper_1101_2678_b200", "libaco_probe.so"))
lib.aco_probe_read_bw_mode.argtypes = [C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
for mib in (12, 24, 48, 64, 96):
    for cg in (0, 1):
        g, ms = C.c_double(), C.c_double()
        rc = lib.aco_probe_read_bw_mode(0, mib << 20, 40, 5, cg, C.byref(g), C.byref(ms))
        print(json.dumps({"mib": mib, "cg": cg, "gbps": round(g.value, 1), "rc": rc}), flush=True)
