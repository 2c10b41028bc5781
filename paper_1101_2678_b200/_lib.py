"""ctypes binding of libaco_gpu.so (include/aco_gpu.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1101_2678_b200/csrc``).  There is no fallback: if the library
is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ACO_GPU_LIB_VARIANT") or os.path.join(HERE, "libaco_gpu.so")

ACO_OK = 0
ACO_E_CUDA = 100
ACO_E_NCCL = 101
ACO_E_UNSUPPORTED = 102
ACO_WIRE_FP64 = 0
ACO_WIRE_FP32 = 1
ACO_WIRE_FIXED64 = 2
ACO_WIRE_MULTIMEM = 3


class aco_gpu_params(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("nn", C.c_int32), ("theta", C.c_int32),
        ("selection", C.c_int32), ("deposit", C.c_int32), ("random_start", C.c_int32),
        ("stream", C.c_int32),
        ("alpha", C.c_double), ("beta", C.c_double), ("rho", C.c_double),
        ("seed", C.c_uint64),
        ("device", C.c_int32),
        ("rank", C.c_int32), ("world", C.c_int32),
        ("ant_begin", C.c_int32), ("ant_end", C.c_int32),
        ("nccl_id", C.c_uint8 * 128),
        ("wire", C.c_int32),
        ("validate_tours", C.c_int32),
    ]


class aco_gpu_iter_record(C.Structure):
    _fields_ = [
        ("iteration", C.c_int32),
        ("best_length", C.c_int64),
        ("mean_length", C.c_double),
        ("construct_ms", C.c_double),
        ("update_ms", C.c_double),
        ("choice_ms", C.c_double),
        ("exchange_ms", C.c_double),
        ("construct_kernel_ms", C.c_double),
        ("ledger", C.c_double * 4),
        ("fallbacks", C.c_int64),
        ("best_so_far", C.c_int64),
        ("certified_fp64", C.c_int64),
    ]


# Every symbol include/aco_gpu.h declares (tests check the export table).
EXPORTS = [
    "aco_errc_name", "aco_parse_instance", "aco_parse_tour", "aco_build_distances",
    "aco_build_nn_lists", "aco_greedy_tour_length", "aco_tour_length",
    "aco_predicted_access_cost", "aco_validate_parameters", "aco_uniform_at", "aco_last_error", "aco_gpu_create", "aco_gpu_destroy",
    "aco_gpu_last_error", "aco_gpu_set_pheromone", "aco_gpu_compute_choice_info",
    "aco_gpu_construct", "aco_gpu_update", "aco_gpu_iterate", "aco_gpu_get_pheromone",
    "aco_gpu_get_choice", "aco_gpu_get_choice32", "aco_gpu_get_topk", "aco_gpu_get_tours", "aco_gpu_get_best",
    "aco_gpu_get_info", "aco_gpu_stream", "aco_gpu_exchange_buffers", "aco_gpu_launch_count", "aco_gpu_describe", "aco_gpu_nccl_unique_id",
    "aco_gpu_philox_uniform", "aco_gpu_validate_tours", "aco_gpu_libm_pow", "aco_gpu_fold",
]

_p = C.c_void_p
_i32 = C.c_int32


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.aco_errc_name.restype = C.c_char_p
    L.aco_errc_name.argtypes = [C.c_int]
    L.aco_last_error.restype = C.c_char_p
    L.aco_parse_instance.argtypes = [C.c_char_p, C.POINTER(_i32), C.POINTER(_i32), _p, _p, _i32,
                                     C.c_char_p, _i32]
    L.aco_parse_tour.argtypes = [C.c_char_p, _p, _i32, C.POINTER(_i32)]
    L.aco_build_distances.argtypes = [_i32, _p, _p, _i32, _p]
    L.aco_build_nn_lists.argtypes = [_i32, _p, _i32, _p]
    L.aco_greedy_tour_length.argtypes = [_i32, _p, C.POINTER(C.c_int64)]
    L.aco_tour_length.argtypes = [_i32, _p, _p, _i32, C.POINTER(C.c_int64)]
    L.aco_predicted_access_cost.argtypes = [_i32, _i32, _i32, _i32, _p]
    L.aco_validate_parameters.argtypes = [C.c_double, C.c_double, C.c_double, _i32, _i32, _i32,
                                          _i32, _i32, _i32]
    L.aco_uniform_at.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
    L.aco_uniform_at.restype = C.c_double
    L.aco_gpu_create.argtypes = [C.POINTER(aco_gpu_params), _p, C.POINTER(_p)]
    L.aco_gpu_destroy.argtypes = [_p]
    L.aco_gpu_destroy.restype = None
    L.aco_gpu_last_error.argtypes = [_p]
    L.aco_gpu_last_error.restype = C.c_char_p
    L.aco_gpu_set_pheromone.argtypes = [_p, _p]
    L.aco_gpu_compute_choice_info.argtypes = [_p]
    L.aco_gpu_construct.argtypes = [_p, C.POINTER(aco_gpu_iter_record)]
    L.aco_gpu_update.argtypes = [_p, C.POINTER(aco_gpu_iter_record)]
    L.aco_gpu_fold.argtypes = [_p, C.POINTER(C.c_int32)]
    L.aco_gpu_iterate.argtypes = [_p, C.POINTER(aco_gpu_iter_record), _p, _p]
    L.aco_gpu_libm_pow.argtypes = [_i32, _i32, _p, _p, _p]
    L.aco_gpu_validate_tours.argtypes = [_p, _p, _p, _i32]
    L.aco_gpu_get_pheromone.argtypes = [_p, _p]
    L.aco_gpu_get_choice.argtypes = [_p, _p]
    L.aco_gpu_get_choice32.argtypes = [_p, _p, _p]
    L.aco_gpu_get_topk.argtypes = [_p, _p, C.POINTER(_i32)]
    L.aco_gpu_get_tours.argtypes = [_p, _p, _p]
    L.aco_gpu_get_best.argtypes = [_p, _p, C.POINTER(C.c_int64)]
    L.aco_gpu_get_info.argtypes = [_p, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32),
                                   C.POINTER(C.c_double), C.POINTER(_i32), C.POINTER(_i32)]
    L.aco_gpu_stream.argtypes = [_p]
    L.aco_gpu_stream.restype = C.c_void_p
    L.aco_gpu_exchange_buffers.argtypes = [_p, C.POINTER(_p), C.POINTER(_p), C.POINTER(_p),
                                           C.POINTER(_p), C.POINTER(_i32), C.POINTER(_i32)]
    L.aco_gpu_launch_count.argtypes = [_p]
    L.aco_gpu_launch_count.restype = C.c_int64
    L.aco_gpu_describe.argtypes = [_p, C.c_char_p, C.c_int32]
    L.aco_gpu_describe.restype = C.c_int32
    L.aco_gpu_nccl_unique_id.argtypes = [_p]
    L.aco_gpu_philox_uniform.argtypes = [_i32, C.c_uint64, C.c_uint32, C.c_uint32, _i32, _p, _p,
                                         _p]
    return L


lib = _load()


def ptr(a: np.ndarray) -> int:
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("buffers passed to libaco_gpu.so must be C-contiguous")
    return a.ctypes.data
