"""Python mirror of the reference's ``aco::`` API (proj/include/aco) over the
B200 engine's C ABI (include/aco_gpu.h, libaco_gpu.so).

Same names, argument meaning and error behaviour as the reference, so code
written against ``aco::Engine`` reads the same here:

    spec    = aco.load_instance("pr2392.tsp")           # tsplib.hpp:281
    problem = aco.build_problem(spec)                   # model.hpp:125
    cfg     = aco.RunConfig(params=aco.Parameters(m=0), # engine.hpp:22
                            selection=aco.SelectionStrategy(aco.Selection.roulette_full),
                            deposit=aco.DepositStrategy(aco.Deposit.accumulate))
    eng     = aco.Engine(problem, cfg)                  # engine.hpp:57
    rec     = eng.run_iteration()                       # engine.hpp:88
    report  = eng.run()                                 # engine.hpp:159

Failures raise ``aco.Error`` carrying an ``Errc`` (errors.hpp:8-40).  Every
device call goes through libaco_gpu.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import lib, ptr


class Errc(enum.IntEnum):  # errors.hpp:8-27
    missing_field = 0
    unsupported_edge_weight_type = 1
    malformed_coord = 2
    dimension_mismatch = 3
    index_out_of_range = 4
    overflow = 5
    invalid_length = 6
    not_a_permutation = 7
    not_closed = 8
    all_visited = 9
    inconsistent_length = 10
    io_error = 11
    config_error = 12


class Error(RuntimeError):
    """aco::Error (errors.hpp:31-40); ``code`` is an Errc, or the raw status
    (ACO_E_CUDA / ACO_E_NCCL / ACO_E_UNSUPPORTED) for engine-side failures."""

    def __init__(self, code, message: str):
        super().__init__(message)
        self.code = code


def _raise(status: int, message: str):
    if 1 <= status <= 13:
        raise Error(Errc(status - 1), message)
    raise Error(status, f"{lib.aco_errc_name(status).decode()}: {message}")


def _check(status: int, ctx=None):
    if status != _lib.ACO_OK:
        msg = (lib.aco_gpu_last_error(ctx) if ctx is not None else lib.aco_last_error()) or b""
        _raise(status, msg.decode(errors="replace"))


class EdgeWeightType(enum.IntEnum):  # tsplib.hpp:16
    euc_2d = 0
    ceil_2d = 1
    att = 2


class Selection(enum.IntEnum):  # construction.hpp:13
    roulette_full = 0
    roulette_nn = 1
    data_parallel_tiled = 2


class Deposit(enum.IntEnum):  # pheromone.hpp:16
    accumulate = 0
    scatter_gather = 1
    scatter_gather_tiled = 2
    symmetric_reduction = 3


class WeightStream(enum.IntEnum):  # include/aco_gpu.h ACO_STREAM_*
    auto = 0
    fp64 = 1
    fp32 = 2


class Wire(enum.IntEnum):  # include/aco_gpu.h ACO_WIRE_*: accumulate arithmetic / delta exchange
    fp64 = 0      # fp64 reds; sharded: fp64 all-reduce
    fp32 = 1      # sharded: fp32 all-reduce (tours may then depend on world)
    fixed64 = 2   # exact int64 fixed-point sums: tau bit-identical for every world
    multimem = 3  # fixed64 through an NVLS multicast object, no collective (world > 1)


def selection_name(s: Selection) -> str:  # construction.hpp:15
    return {Selection.roulette_full: "roulette", Selection.roulette_nn: "nn",
            Selection.data_parallel_tiled: "data-parallel"}[Selection(s)]


def deposit_name(d: Deposit) -> str:  # pheromone.hpp:18
    return {Deposit.accumulate: "accumulate", Deposit.scatter_gather: "scatter-gather",
            Deposit.scatter_gather_tiled: "scatter-gather-tiled",
            Deposit.symmetric_reduction: "symmetric-reduction"}[Deposit(d)]


# ---- instances (tsplib.hpp) --------------------------------------------
@dataclass
class InstanceSpec:  # tsplib.hpp:27-32
    name: str = ""
    dimension: int = 0
    edge_weight_type: EdgeWeightType = EdgeWeightType.euc_2d
    xs: np.ndarray = field(default_factory=lambda: np.zeros(0))
    ys: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @property
    def coords(self):
        return list(zip(self.xs.tolist(), self.ys.tolist()))


def parse_instance(text: str) -> InstanceSpec:  # tsplib.hpp:76
    raw = text.encode()
    dim, ewt = C.c_int32(), C.c_int32()
    _check(lib.aco_parse_instance(raw, C.byref(dim), C.byref(ewt), None, None, 0, None, 0))
    xs = np.zeros(dim.value, np.float64)
    ys = np.zeros(dim.value, np.float64)
    name = C.create_string_buffer(4096)
    _check(lib.aco_parse_instance(raw, C.byref(dim), C.byref(ewt), ptr(xs), ptr(ys), dim.value,
                                  name, 4096))
    return InstanceSpec(name.value.decode(), dim.value, EdgeWeightType(ewt.value), xs, ys)


def load_instance(path: str) -> InstanceSpec:  # tsplib.hpp:272-283
    try:
        with open(path, "rb") as f:
            text = f.read().decode("latin-1")
    except OSError:
        raise Error(Errc.io_error, "cannot open file: " + path) from None
    return parse_instance(text)


def parse_tour(text: str) -> np.ndarray:  # tsplib.hpp:238
    cap = max(16, text.count("\n") * 16 + 16)
    out = np.zeros(cap, np.int32)
    ln = C.c_int32()
    _check(lib.aco_parse_tour(text.encode(), ptr(out), cap, C.byref(ln)))
    return out[: ln.value].copy()


def synthetic_instance(n: int, seed_state: int = 42) -> InstanceSpec:
    """Uniform EUC_2D instance of SURVEY.md App. B: splitmix64 seeded with
    42, integer coordinates in [0, 10000], x before y."""
    mask = (1 << 64) - 1
    s = seed_state
    xs = np.zeros(n, np.float64)
    ys = np.zeros(n, np.float64)

    def nxt():
        nonlocal s
        s = (s + 0x9E3779B97F4A7C15) & mask
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        return z ^ (z >> 31)

    for i in range(n):
        xs[i] = nxt() % 10001
        ys[i] = nxt() % 10001
    return InstanceSpec(f"synth{n}", n, EdgeWeightType.euc_2d, xs, ys)


# ---- model (model.hpp) ---------------------------------------------------
@dataclass
class ProblemInstance:  # model.hpp:23-27 (the heuristic is folded into the device table)
    n: int
    dist: np.ndarray  # int32 n x n


def build_problem(spec: InstanceSpec) -> ProblemInstance:  # model.hpp:125
    n = spec.dimension
    d = np.zeros((n, n), np.int32)
    _check(lib.aco_build_distances(n, ptr(np.ascontiguousarray(spec.xs, np.float64)),
                                   ptr(np.ascontiguousarray(spec.ys, np.float64)),
                                   int(spec.edge_weight_type), ptr(d)))
    return ProblemInstance(n, d)


def build_nn_lists(problem: ProblemInstance, nn: int) -> np.ndarray:  # model.hpp:177
    out = np.zeros((problem.n, nn), np.int32)
    _check(lib.aco_build_nn_lists(problem.n, ptr(problem.dist), nn, ptr(out)))
    return out


def tour_length(problem: ProblemInstance, tour) -> int:  # model.hpp:205
    t = np.ascontiguousarray(tour, np.int32)
    out = C.c_int64()
    _check(lib.aco_tour_length(problem.n, ptr(problem.dist), ptr(t), len(t), C.byref(out)))
    return out.value


def greedy_nn_tour_length(problem: ProblemInstance) -> int:  # model.hpp:230
    out = C.c_int64()
    _check(lib.aco_greedy_tour_length(problem.n, ptr(problem.dist), C.byref(out)))
    return out.value


def initial_pheromone(problem: ProblemInstance, m: int) -> float:  # model.hpp:258 (tau0 value)
    return float(m) / float(greedy_nn_tour_length(problem))


@dataclass
class Parameters:  # model.hpp:29-53
    alpha: float = 1.0
    beta: float = 2.0
    rho: float = 0.5
    m: int = 0
    nn: int = 30
    iterations: int = 100
    seed: int = 1
    tile_size: int = 64


@dataclass
class SelectionStrategy:  # construction.hpp:24-27
    variant: Selection = Selection.roulette_nn
    tile_size: int = 64


@dataclass
class DepositStrategy:  # pheromone.hpp:28-31
    variant: Deposit = Deposit.accumulate
    tile_size: int = 64


@dataclass
class AccessLedger:  # pheromone.hpp:37-54
    global_loads: float = 0.0
    global_stores: float = 0.0
    shared_loads: float = 0.0
    atomic_ops: float = 0.0


def predicted_access_cost(strategy: DepositStrategy, n: int, m: int, theta: int) -> AccessLedger:
    out = np.zeros(4, np.float64)  # pheromone.hpp:366
    _check(lib.aco_predicted_access_cost(int(strategy.variant), n, m, theta, ptr(out)))
    return AccessLedger(*out.tolist())


@dataclass
class RunConfig:  # engine.hpp:22-29 (+ device placement)
    params: Parameters = field(default_factory=Parameters)
    selection: SelectionStrategy = field(default_factory=SelectionStrategy)
    deposit: DepositStrategy = field(default_factory=DepositStrategy)
    workers: int = 0  # accepted for API compatibility; the grid replaces the pool
    random_start: bool = False
    instance_path: str = ""
    device: int = 0
    stream: WeightStream = WeightStream.auto
    rank: int = 0
    world: int = 1
    ant_begin: int = 0
    ant_end: int = 0
    nccl_id: Optional[bytes] = None
    wire: Wire = Wire.fp64  # fp32 halves the all-reduce; tours then depend on world
    validate_tours: bool = False  # debug: device tour validation after every construction


@dataclass
class IterationRecord:  # engine.hpp:31-38 (+ device detail)
    iteration: int = 0
    best_length: int = 0
    mean_length: float = 0.0
    construct_ms: float = 0.0
    update_ms: float = 0.0
    deposit_ledger: AccessLedger = field(default_factory=AccessLedger)
    choice_ms: float = 0.0
    exchange_ms: float = 0.0
    construct_kernel_ms: float = 0.0
    fallbacks: int = 0
    best_so_far: int = 0
    certified_fp64: int = 0


@dataclass
class RunReport:  # engine.hpp:40-47
    instance_name: str = ""
    n: int = 0
    m: int = 0
    seed: int = 0
    config: Optional[RunConfig] = None
    best_tour: Optional[np.ndarray] = None
    best_length: int = 0
    per_iteration: List[IterationRecord] = field(default_factory=list)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib.aco_gpu_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Engine:
    """aco::Engine (engine.hpp:55-196) on one B200.

    The colony state (tau, choice, tours) lives on the device; the accessors
    copy it out on demand.  With ``config.world > 1`` this engine is one rank
    of an ant-sharded colony."""

    def __init__(self, problem: ProblemInstance, config: RunConfig):
        self._problem = problem
        self._config = config
        p = _lib.aco_gpu_params()
        prm = config.params
        p.n = problem.n
        p.m = prm.m
        p.nn = prm.nn
        p.theta = prm.tile_size
        p.selection = int(config.selection.variant)
        p.deposit = int(config.deposit.variant)
        p.random_start = int(bool(config.random_start))
        p.stream = int(config.stream)
        p.alpha, p.beta, p.rho = prm.alpha, prm.beta, prm.rho
        p.seed = prm.seed & ((1 << 64) - 1)
        p.device = config.device
        p.rank, p.world = config.rank, config.world
        p.ant_begin, p.ant_end = config.ant_begin, config.ant_end
        if config.nccl_id is not None:
            C.memmove(p.nccl_id, config.nccl_id, 128)
        p.wire = int(config.wire)
        p.validate_tours = int(bool(config.validate_tours))
        if prm.iterations < 1:
            raise Error(Errc.config_error, "iterations must be >= 1")
        h = C.c_void_p()
        dist = np.ascontiguousarray(problem.dist, np.int32)
        _check(lib.aco_gpu_create(C.byref(p), ptr(dist), C.byref(h)))
        self._h = h
        m, a0, a1, st, it = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        tau0 = C.c_double()
        lib.aco_gpu_get_info(h, C.byref(m), C.byref(a0), C.byref(a1), C.byref(tau0), C.byref(st),
                             C.byref(it))
        self.m = m.value
        self.ant_begin, self.ant_end = a0.value, a1.value
        self.tau0 = tau0.value
        self.weight_stream = WeightStream(st.value)
        self._n = problem.n

    def close(self):
        if getattr(self, "_h", None):
            lib.aco_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- accessors (engine.hpp:79-86)
    def problem(self) -> ProblemInstance:
        return self._problem

    def config(self) -> RunConfig:
        return self._config

    def pheromone(self) -> np.ndarray:
        out = np.zeros((self._n, self._n), np.float64)
        _check(lib.aco_gpu_get_pheromone(self._h, ptr(out)), self._h)
        return out

    def choice(self) -> np.ndarray:
        out = np.zeros((self._n, self._n), np.float64)
        _check(lib.aco_gpu_get_choice(self._h, ptr(out)), self._h)
        return out

    def choice32(self):
        out = np.zeros((self._n, self._n), np.float32)
        sc = np.zeros(self._n, np.int32)
        _check(lib.aco_gpu_get_choice32(self._h, ptr(out), ptr(sc)), self._h)
        return out, sc

    def topk(self) -> np.ndarray:
        """nn selection's per-row argmax cache [n, K] (diagnostic; see
        aco_gpu_get_topk)."""
        k = C.c_int32(0)
        _check(lib.aco_gpu_get_topk(self._h, None, C.byref(k)), self._h)
        out = np.zeros((self._n, k.value), np.int32)
        _check(lib.aco_gpu_get_topk(self._h, ptr(out), None), self._h)
        return out

    def ants(self):
        """(tours[m_local, n+1], lengths[m_local]) of the last construction."""
        k = self.ant_end - self.ant_begin
        t = np.zeros((k, self._n + 1), np.int32)
        l = np.zeros(k, np.int64)
        _check(lib.aco_gpu_get_tours(self._h, ptr(t), ptr(l)), self._h)
        return t, l

    def best_length(self) -> int:
        ln = C.c_int64()
        _check(lib.aco_gpu_get_best(self._h, None, C.byref(ln)), self._h)
        return ln.value

    def best_tour(self) -> np.ndarray:
        t = np.zeros(self._n + 1, np.int32)
        ln = C.c_int64()
        _check(lib.aco_gpu_get_best(self._h, ptr(t), C.byref(ln)), self._h)
        return t

    def validate_tours(self, tours: np.ndarray, lengths: np.ndarray):
        """TourBuffer::make's checks (pheromone.hpp:67-90) on the device: raises
        Error(not_closed | not_a_permutation | inconsistent_length)."""
        t = np.ascontiguousarray(tours, np.int32)
        ln = np.ascontiguousarray(lengths, np.int64)
        if t.ndim != 2 or t.shape[1] != self._n + 1 or ln.shape != (t.shape[0],):
            raise Error(Errc.invalid_length, "tours must be (count, n+1) with count lengths")
        _check(lib.aco_gpu_validate_tours(self._h, ptr(t), ptr(ln), t.shape[0]), self._h)

    def set_pheromone(self, tau: np.ndarray):
        t = np.ascontiguousarray(tau, np.float64)
        _check(lib.aco_gpu_set_pheromone(self._h, ptr(t)), self._h)

    def compute_choice_info(self):
        _check(lib.aco_gpu_compute_choice_info(self._h), self._h)

    def stream_handle(self) -> int:
        """cudaStream_t of this engine (for CUDA-event timing on the launching stream)."""
        return lib.aco_gpu_stream(self._h)

    def exchange_buffers(self):
        """Device pointers of the shard exchange buffers (aco_gpu_exchange_buffers)."""
        ps = [C.c_void_p() for _ in range(4)]
        S, P64 = C.c_int32(), C.c_int32()
        _check(lib.aco_gpu_exchange_buffers(self._h, *[C.byref(x) for x in ps], C.byref(S),
                                            C.byref(P64)), self._h)
        return {"succ": ps[0].value, "pred": ps[1].value, "inv": ps[2].value,
                "delta": ps[3].value, "S": S.value, "P64": P64.value}

    def launch_count(self) -> int:
        return lib.aco_gpu_launch_count(self._h)

    def describe(self) -> str:
        """Kernel name and launch shape of the last construction (diagnostics)."""
        import ctypes
        buf = ctypes.create_string_buffer(256)
        lib.aco_gpu_describe(self._h, buf, 256)
        return buf.value.decode()

    # -- the iteration (engine.hpp:88-157)
    @staticmethod
    def _record(r: _lib.aco_gpu_iter_record) -> IterationRecord:
        return IterationRecord(r.iteration, r.best_length, r.mean_length, r.construct_ms,
                               r.update_ms, AccessLedger(*list(r.ledger)), r.choice_ms,
                               r.exchange_ms, r.construct_kernel_ms, r.fallbacks, r.best_so_far,
                               r.certified_fp64)

    def construct(self) -> IterationRecord:
        r = _lib.aco_gpu_iter_record()
        _check(lib.aco_gpu_construct(self._h, C.byref(r)), self._h)
        return self._record(r)

    def fold(self) -> int:
        """Row-sharded gather deposit, external-exchange mode (aco_gpu_fold):
        folds this rank's row block into the delta rows; returns the block
        size B (rows [rank*B, rank*B+B))."""
        b = C.c_int32()
        _check(lib.aco_gpu_fold(self._h, C.byref(b)), self._h)
        return b.value

    def update(self) -> IterationRecord:
        r = _lib.aco_gpu_iter_record()
        _check(lib.aco_gpu_update(self._h, C.byref(r)), self._h)
        return self._record(r)

    def _check_out(self, a: Optional[np.ndarray], dtype, shape, name: str):
        # the C side writes exactly mloc*(n+1) int32 / mloc int64: anything else
        # would overrun (or be misread from) the caller's host buffer
        if a is None:
            return
        if a.dtype != dtype or tuple(a.shape) != shape or not a.flags["C_CONTIGUOUS"] \
                or not a.flags["WRITEABLE"]:
            raise Error(Errc.dimension_mismatch,
                        f"{name} must be a writeable C-contiguous {np.dtype(dtype).name} array "
                        f"of shape {shape} (this context's ants), got {a.dtype} {a.shape}")

    def run_iteration(self, tours_out: Optional[np.ndarray] = None,
                      lengths_out: Optional[np.ndarray] = None) -> IterationRecord:
        k = self.ant_end - self.ant_begin
        self._check_out(tours_out, np.int32, (k, self._n + 1), "tours_out")
        self._check_out(lengths_out, np.int64, (k,), "lengths_out")
        r = _lib.aco_gpu_iter_record()
        _check(lib.aco_gpu_iterate(self._h, C.byref(r),
                                   None if tours_out is None else ptr(tours_out),
                                   None if lengths_out is None else ptr(lengths_out)), self._h)
        return self._record(r)

    def run(self) -> RunReport:  # engine.hpp:159-171
        rep = RunReport(n=self._n, m=self.m, seed=self._config.params.seed, config=self._config)
        for _ in range(self._config.params.iterations):
            rep.per_iteration.append(self.run_iteration())
        rep.best_length = self.best_length()
        rep.best_tour = self.best_tour()
        return rep


def run(config: RunConfig) -> RunReport:  # engine.hpp:198-204
    spec = load_instance(config.instance_path)
    with Engine(build_problem(spec), config) as eng:
        rep = eng.run()
    rep.instance_name = spec.name
    return rep


@dataclass
class MatrixDiff:  # pheromone.hpp:400-404
    max_abs_diff: float = 0.0
    i: int = 0
    j: int = 0


def max_cell_difference(a: np.ndarray, b: np.ndarray) -> MatrixDiff:  # pheromone.hpp:406
    d = np.abs(a - b)
    k = int(np.argmax(d))
    if d.flat[k] <= 0.0:
        return MatrixDiff()
    return MatrixDiff(float(d.flat[k]), k // a.shape[1], k % a.shape[1])


@dataclass
class VerifyReport:  # engine.hpp:208-225
    strategies: list = field(default_factory=list)  # (variant, ledger, predicted, ok)
    pairs: list = field(default_factory=list)       # (a, b, MatrixDiff, pass)
    all_pass: bool = False


def verify_deposit_equivalence(problem: ProblemInstance, config: RunConfig,
                               tolerance: float = 1e-9) -> VerifyReport:
    """engine.hpp:227-292 on the GPU: one iteration-0 construction (identical
    in every engine: the draws are keyed by (seed, iteration, ant, step)),
    then each deposit variant from the same tau0; ``all_pass`` = every
    pairwise max cell difference <= tolerance.

    Ledgers: the reference COUNTS the abstract accesses its CPU loops make
    and compares them with the closed form.  The device kernels make no such
    accesses, so the engine reports the closed-form model itself
    (predicted_access_cost); each strategy entry carries it with ok=True by
    construction, and the ledger is NOT part of ``all_pass`` here (a
    measured-vs-predicted ledger check runs against the reference harness
    in tests/test_abi.py)."""
    variants = [Deposit.accumulate, Deposit.scatter_gather, Deposit.scatter_gather_tiled,
                Deposit.symmetric_reduction]
    results, rep = [], VerifyReport()
    tours0 = None
    for v in variants:
        cfg = RunConfig(params=config.params, selection=config.selection,
                        deposit=DepositStrategy(v, config.params.tile_size),
                        random_start=False, device=config.device, stream=config.stream)
        with Engine(problem, cfg) as eng:
            rec = eng.run_iteration()
            t, _ = eng.ants()
            if tours0 is None:
                tours0 = t
            elif not np.array_equal(t, tours0):
                raise Error(Errc.inconsistent_length, "engines built different tours")
            results.append(eng.pheromone())
            pred = predicted_access_cost(cfg.deposit, problem.n, eng.m, config.params.tile_size)
            rep.strategies.append((v, rec.deposit_ledger, pred, True))
    rep.all_pass = True
    for a in range(len(variants)):
        for b in range(a + 1, len(variants)):
            d = max_cell_difference(results[a], results[b])
            ok = d.max_abs_diff <= tolerance
            rep.pairs.append((variants[a], variants[b], d, ok))
            rep.all_pass = rep.all_pass and ok
    return rep


def philox_uniform_device(seed: int, iteration: int, ant: int, steps, draws, device: int = 0):
    """Device Philox draws (rng.hpp:74-80) for unit parity tests."""
    st = np.ascontiguousarray(steps, np.uint32)
    dr = np.ascontiguousarray(draws, np.uint32)
    out = np.zeros(len(st), np.float64)
    _check(lib.aco_gpu_philox_uniform(device, seed, iteration, ant, len(st), ptr(st), ptr(dr),
                                      ptr(out)))
    return out
