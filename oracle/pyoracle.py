"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU oracle.

Two checkers live here:

* ``Oracle``    -> oracle/_build/libaco_oracle.so, the plain-C restatement
                  (oracle/aco_oracle.c), built by ``make -C oracle``.
* ``Reference`` -> oracle/_ref/libaco_ref.so, the reference's own headers
                  compiled unmodified (oracle/ref_harness.cpp), built by
                  ``make -C oracle ref`` where /root/reference exists; the
                  prebuilt .so travels to the GPU box.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference /
cpu_baseline legs may import this module.  The product package
(paper_1101_2678_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libaco_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libaco_ref.so")
REF_INC = "/root/reference/proj/include"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """Compile the checker(s). ``ref=None`` builds _ref only if /root/reference exists."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref or (ref is None and os.path.isdir(REF_INC)):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def synth_coords(n: int, state: int = 42):
    o = Oracle.get()
    xs = np.zeros(n, np.float64)
    ys = np.zeros(n, np.float64)
    o.lib.orc_synth_coords(n, C.c_uint64(state), xs, ys)
    return xs, ys


class Oracle:
    _inst = None

    @classmethod
    def get(cls) -> "Oracle":
        if cls._inst is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            cls._inst = cls(ORACLE_SO)
        return cls._inst

    def __init__(self, path: str):
        L = C.CDLL(path)
        self.lib = L
        L.orc_philox.argtypes = [_u32p, C.c_uint64, _u32p]
        L.orc_uniform_at.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_uniform_at.restype = C.c_double
        L.orc_synth_coords.argtypes = [C.c_int, C.c_uint64, _f64p, _f64p]
        L.orc_build_dist.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p]
        L.orc_greedy_nn_tour_length.argtypes = [C.c_int, _i32p]
        L.orc_greedy_nn_tour_length.restype = C.c_int64
        L.orc_tau0.argtypes = [C.c_int, _i32p, C.c_int]
        L.orc_tau0.restype = C.c_double
        L.orc_build_nn_lists.argtypes = [C.c_int, _i32p, C.c_int, _i32p]
        L.orc_choice_info.argtypes = [C.c_int, _i32p, _f64p, C.c_double, C.c_double, _f64p]
        L.orc_tour_length.argtypes = [C.c_int, _i32p, _i32p]
        L.orc_tour_length.restype = C.c_int64
        L.orc_construct.argtypes = [C.c_int, _i32p, _f64p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                    C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_int, _i32p,
                                    _i64p, _i64p]
        L.orc_update.argtypes = [C.c_int, C.c_int, _i32p, _i64p, C.c_double, C.c_int, _f64p]
        L.orc_pow.argtypes = [C.c_int, _f64p, _f64p, _f64p]

    # -- rng.hpp
    def philox(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.lib.orc_philox(np.asarray(ctr, np.uint32), C.c_uint64(key), out)
        return out

    def uniform_at(self, seed, it, ant, step, draw):
        return self.lib.orc_uniform_at(seed, it, ant, step, draw)

    # -- model.hpp
    def build_dist(self, xs, ys, ewt=0):
        n = len(xs)
        d = np.zeros((n, n), np.int32)
        rc = self.lib.orc_build_dist(n, np.ascontiguousarray(xs, np.float64),
                                     np.ascontiguousarray(ys, np.float64), ewt, d)
        if rc:
            raise RuntimeError(f"orc_build_dist rc={rc}")
        return d

    def tau0(self, dist, m):
        return self.lib.orc_tau0(dist.shape[0], dist, m)

    def greedy(self, dist):
        return self.lib.orc_greedy_nn_tour_length(dist.shape[0], dist)

    def nn_lists(self, dist, nn):
        n = dist.shape[0]
        out = np.zeros((n, nn), np.int32)
        rc = self.lib.orc_build_nn_lists(n, dist, nn, out)
        if rc:
            raise RuntimeError(f"orc_build_nn_lists rc={rc}")
        return out

    def choice(self, dist, tau, alpha=1.0, beta=2.0):
        n = dist.shape[0]
        out = np.zeros((n, n), np.float64)
        self.lib.orc_choice_info(n, dist, np.ascontiguousarray(tau), alpha, beta, out)
        return out

    def pow(self, x, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(np.broadcast_to(y, x.shape), np.float64)
        out = np.zeros_like(x)
        self.lib.orc_pow(len(x), x, y, out)
        return out

    def tour_length(self, dist, tour):
        return self.lib.orc_tour_length(dist.shape[0], dist, np.ascontiguousarray(tour, np.int32))

    # -- construction.hpp
    def construct(self, dist, choice, seed, iteration, k0, k1, selection=0, nn_lists=None,
                  theta=64, random_start=False):
        n = dist.shape[0]
        cnt = k1 - k0
        tours = np.zeros((cnt, n + 1), np.int32)
        lens = np.zeros(cnt, np.int64)
        stats = np.zeros(3, np.int64)
        nnp = None
        nn = 0
        if nn_lists is not None:
            nn_lists = np.ascontiguousarray(nn_lists, np.int32)
            nnp = nn_lists.ctypes.data
            nn = nn_lists.shape[1]
        rc = self.lib.orc_construct(n, dist, np.ascontiguousarray(choice), nnp, nn, selection,
                                    theta, C.c_uint64(seed), iteration, int(random_start), k0, k1,
                                    tours, lens, stats)
        if rc:
            raise RuntimeError(f"orc_construct rc={rc}")
        return tours, lens, stats

    # -- pheromone.hpp
    def update(self, tau, tours, lengths, rho, deposit):
        t = np.array(tau, np.float64, copy=True, order="C")
        m = tours.shape[0]
        n = tours.shape[1] - 1
        self.lib.orc_update(n, m, np.ascontiguousarray(tours, np.int32),
                            np.ascontiguousarray(lengths, np.int64), rho, deposit, t)
        return t


class Reference:
    """The reference's own C++ (headers compiled unmodified) behind a C shim."""

    _inst = None

    @classmethod
    def get(cls) -> "Reference":
        if cls._inst is None:
            if not os.path.exists(REF_SO):
                if os.path.isdir(REF_INC):
                    build(ref=True)
                else:
                    raise FileNotFoundError(REF_SO)
            cls._inst = cls(REF_SO)
        return cls._inst

    def __init__(self, path: str):
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_philox_block.argtypes = [C.c_uint32] * 4 + [C.c_uint64, _u32p]
        L.ref_uniform_at.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_uniform_at.restype = C.c_double
        L.ref_parse_instance.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.c_void_p, C.c_void_p, C.c_int]
        L.ref_parse_tour.argtypes = [C.c_char_p, _i32p, C.c_int, C.POINTER(C.c_int)]
        L.ref_build_problem.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, C.c_void_p]
        L.ref_compute_choice_info.argtypes = [C.c_int, _i32p, _f64p, C.c_double, C.c_double,
                                              _f64p]
        L.ref_build_nn_lists.argtypes = [C.c_int, _i32p, C.c_int, _i32p]
        L.ref_tour_length.argtypes = [C.c_int, _i32p, _i32p, C.c_int, C.POINTER(C.c_int64)]
        L.ref_initial_pheromone.argtypes = [C.c_int, _i32p, C.c_int, C.POINTER(C.c_double)]
        L.ref_construct.argtypes = [C.c_int, _i32p, _f64p, C.c_void_p, C.c_int, C.c_int,
                                    C.c_int, C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                    _i32p, _i64p]
        L.ref_update.argtypes = [C.c_int, _i32p, C.c_int, _i32p, _i64p, C.c_double, C.c_int,
                                 C.c_int, C.c_int, _f64p, C.c_void_p]
        L.ref_predicted_access_cost.argtypes = [C.c_int] * 4 + [_f64p]
        L.ref_engine_create.argtypes = [C.c_int, _f64p, _f64p, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p)]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_m.argtypes = [C.c_void_p]
        L.ref_engine_workers.argtypes = [C.c_void_p]
        L.ref_engine_iterate.argtypes = [C.c_void_p, _f64p]
        L.ref_engine_tau.argtypes = [C.c_void_p, _f64p]
        L.ref_engine_choice.argtypes = [C.c_void_p, _f64p]
        L.ref_engine_tours.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_engine_best.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_engine_best.restype = C.c_int64
        L.ref_verify_deposit_equivalence.argtypes = [C.c_int, _f64p, _f64p, C.c_int, C.c_int,
                                                     C.c_int, C.c_int, C.c_int, C.c_uint64,
                                                     C.c_double, C.POINTER(C.c_int),
                                                     C.POINTER(C.c_double)]

    def format_double(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        self.lib.ref_format_double.argtypes = [C.c_double, C.c_char_p]
        self.lib.ref_format_double(v, buf)
        return buf.value.decode()

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"reference rc={rc}: {self.lib.ref_last_error().decode()}")

    def philox(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.lib.ref_philox_block(*[int(c) for c in ctr], C.c_uint64(key), out)
        return out

    def uniform_at(self, seed, it, ant, step, draw):
        return self.lib.ref_uniform_at(seed, it, ant, step, draw)

    def parse_instance(self, text: str):
        dim, ewt = C.c_int(), C.c_int()
        self._check(self.lib.ref_parse_instance(text.encode(), C.byref(dim), C.byref(ewt),
                                                None, None, 0))
        xs = np.zeros(dim.value, np.float64)
        ys = np.zeros(dim.value, np.float64)
        self._check(self.lib.ref_parse_instance(text.encode(), C.byref(dim), C.byref(ewt),
                                                xs.ctypes.data, ys.ctypes.data, dim.value))
        return xs, ys, ewt.value

    def parse_tour(self, text: str, cap: int = 1 << 20):
        out = np.zeros(cap, np.int32)
        ln = C.c_int()
        self._check(self.lib.ref_parse_tour(text.encode(), out, cap, C.byref(ln)))
        return out[: ln.value].copy()

    def build_problem(self, xs, ys, ewt=0):
        n = len(xs)
        d = np.zeros((n, n), np.int32)
        self._check(self.lib.ref_build_problem(n, np.ascontiguousarray(xs, np.float64),
                                               np.ascontiguousarray(ys, np.float64), ewt, d,
                                               None))
        return d

    def choice(self, dist, tau, alpha=1.0, beta=2.0):
        n = dist.shape[0]
        out = np.zeros((n, n), np.float64)
        self._check(self.lib.ref_compute_choice_info(n, dist, np.ascontiguousarray(tau), alpha,
                                                     beta, out))
        return out

    def nn_lists(self, dist, nn):
        n = dist.shape[0]
        out = np.zeros((n, nn), np.int32)
        self._check(self.lib.ref_build_nn_lists(n, dist, nn, out))
        return out

    def tour_length(self, dist, tour):
        out = C.c_int64()
        t = np.ascontiguousarray(tour, np.int32)
        self._check(self.lib.ref_tour_length(dist.shape[0], dist, t, len(t), C.byref(out)))
        return out.value

    def tau0(self, dist, m):
        out = C.c_double()
        self._check(self.lib.ref_initial_pheromone(dist.shape[0], dist, m, C.byref(out)))
        return out.value

    def construct(self, dist, choice, seed, iteration, k0, k1, selection=0, nn_lists=None,
                  theta=64, random_start=False):
        n = dist.shape[0]
        tours = np.zeros((k1 - k0, n + 1), np.int32)
        lens = np.zeros(k1 - k0, np.int64)
        nnp, nn = None, 0
        if nn_lists is not None:
            nn_lists = np.ascontiguousarray(nn_lists, np.int32)
            nnp, nn = nn_lists.ctypes.data, nn_lists.shape[1]
        self._check(self.lib.ref_construct(n, dist, np.ascontiguousarray(choice), nnp, nn,
                                           selection, theta, C.c_uint64(seed), iteration,
                                           int(random_start), k0, k1, tours, lens))
        return tours, lens

    def update(self, dist, tau, tours, lengths, rho, deposit, theta=64, workers=1):
        t = np.array(tau, np.float64, copy=True, order="C")
        led = np.zeros(4, np.float64)
        self._check(self.lib.ref_update(dist.shape[0], dist, tours.shape[0],
                                        np.ascontiguousarray(tours, np.int32),
                                        np.ascontiguousarray(lengths, np.int64), rho, deposit,
                                        theta, workers, t, led.ctypes.data))
        return t, led

    def predicted_access_cost(self, deposit, n, m, theta):
        out = np.zeros(4, np.float64)
        self.lib.ref_predicted_access_cost(deposit, n, m, theta, out)
        return out


class RefEngine:
    """aco::Engine (engine.hpp:55-196) driven through the harness."""

    def __init__(self, xs, ys, ewt=0, alpha=1.0, beta=2.0, rho=0.5, m=0, nn=30, seed=1,
                 theta=64, selection=0, deposit=0, workers=0, random_start=False):
        self.ref = Reference.get()
        self.n = len(xs)
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_engine_create(
            self.n, np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64),
            ewt, alpha, beta, rho, m, nn, C.c_uint64(seed), theta, selection, deposit, workers,
            int(random_start), C.byref(h)))
        self.h = h
        self.m = self.ref.lib.ref_engine_m(h)
        self.workers = self.ref.lib.ref_engine_workers(h)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_engine_destroy(self.h)
            self.h = None

    def run_iteration(self):
        rec = np.zeros(6, np.float64)
        self.ref._check(self.ref.lib.ref_engine_iterate(self.h, rec))
        return {"best_length": int(rec[0]), "mean_length": rec[1], "construct_ms": rec[2],
                "update_ms": rec[3], "choice_ms": rec[4], "atomic_ops": rec[5]}

    def pheromone(self):
        out = np.zeros((self.n, self.n), np.float64)
        self.ref.lib.ref_engine_tau(self.h, out)
        return out

    def choice(self):
        out = np.zeros((self.n, self.n), np.float64)
        self.ref.lib.ref_engine_choice(self.h, out)
        return out

    def tours(self):
        t = np.zeros((self.m, self.n + 1), np.int32)
        l = np.zeros(self.m, np.int64)
        self.ref.lib.ref_engine_tours(self.h, t.ctypes.data, l.ctypes.data)
        return t, l

    def best(self):
        t = np.zeros(self.n + 1, np.int32)
        ln = self.ref.lib.ref_engine_best(self.h, t.ctypes.data)
        return ln, t


def fnv1a64(arr: np.ndarray) -> str:
    """FNV-1a-64 over the raw little-endian bytes (SURVEY.md App. B hashes)."""
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(arr).tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
