"""Cluster / DSMEM latencies on this B200 (libaco_probe.so aco_probe_cluster):
the per-step cost a thread-block-cluster-per-ant roulette would pay.
    python tools/cluster_probe.py"""
import ctypes as C
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "paper_1101_2678_b200", "libaco_probe.so"))
L.aco_probe_cluster.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
out = {}
for name, K, mode in (("dsmem_round_trip_k2", 2, 0), ("cluster_sync_k2", 2, 1), ("cluster_sync_k4", 4, 1),
                      ("cluster_sync_k8", 8, 1), ("step_exchange_k2", 2, 2), ("step_exchange_k4", 4, 2),
                      ("step_exchange_k8", 8, 2)):
    v = C.c_double()
    rc = L.aco_probe_cluster(0, K, mode, 20000, C.byref(v))
    out[name] = round(v.value, 1) if rc == 0 else f"rc={rc}"
print(json.dumps({"cycles": out}))
