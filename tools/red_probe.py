"""Atomic (red.global.add.f64) throughput at random addresses vs buffer size:
the roofline denominator of k_deposit_atomic (libaco_probe.so aco_probe_red)."""
import ctypes as C
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def measure(device=0):
    L = C.CDLL(os.path.join(ROOT, "paper_1101_2678_b200", "libaco_probe.so"))
    L.aco_probe_red.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_int,
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]
    out = {}
    for mb in (46, 800):
        g, ms = C.c_double(), C.c_double()
        rc = L.aco_probe_red(device, mb << 20, 200_000_000 if mb > 100 else 50_000_000, 3,
                             C.byref(g), C.byref(ms))
        out[f"red_f64_random_{mb}MB_gops"] = round(g.value, 1) if rc == 0 else None
    return out


if __name__ == "__main__":
    print(json.dumps(measure()))
