"""Dependent-chain latencies (cycles/op) of FP64/FP32/shuffle on this GPU."""
import ctypes as C, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "paper_1101_2678_b200", "libaco_probe.so"))
L.aco_probe_latency.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for op, name in enumerate(["DADD", "DMUL", "DFMA", "FADD", "F2F+FADD+F2F", "SHFL.f64+DADD", "SHFL.f32", "DSETP+DADD/select"]):
    v = C.c_double()
    L.aco_probe_latency(0, op, 2000, C.byref(v))
    print(f"{name:20s} {v.value:8.2f} cycles/op")
