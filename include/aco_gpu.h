/* aco_gpu.h — C ABI of the B200-native Ant System engine (libaco_gpu.so).
 *
 * Drop-in boundary for the reference's iteration loop.  The reference is a
 * header-only C++20 library with no FFI; its "operator API" is the aco::
 * surface in proj/include/aco.  Each entry point below names the reference
 * function(s) it replaces (paths relative to /root/reference/proj):
 *
 *   aco_parse_instance      <- aco::parse_instance        include/aco/tsplib.hpp:76
 *   aco_build_distances     <- aco::build_problem         include/aco/model.hpp:125
 *                              (dist part; edge_weight tsplib.hpp:190)
 *   aco_build_nn_lists      <- aco::build_nn_lists        include/aco/model.hpp:177
 *   aco_greedy_tour_length  <- aco::greedy_nn_tour_length include/aco/model.hpp:230
 *   aco_tour_length         <- aco::tour_length           include/aco/model.hpp:205
 *   aco_predicted_access_cost <- aco::predicted_access_cost include/aco/pheromone.hpp:366
 *   aco_gpu_create          <- aco::Engine::Engine        include/aco/engine.hpp:57-79
 *   aco_gpu_compute_choice_info <- aco::compute_choice_info include/aco/model.hpp:154
 *   aco_gpu_construct       <- the construction fork       include/aco/engine.hpp:95-129
 *                              (construct_tour construction.hpp:181, select_next :164)
 *   aco_gpu_update          <- evaporate + apply_deposit + compute_choice_info
 *                              + best-so-far              include/aco/engine.hpp:131-155
 *   aco_gpu_iterate         <- aco::Engine::run_iteration include/aco/engine.hpp:88
 *   aco_gpu_get_pheromone   <- aco::Engine::pheromone     include/aco/engine.hpp:82
 *   aco_gpu_get_choice      <- aco::Engine::choice        include/aco/engine.hpp:83
 *   aco_gpu_get_tours       <- aco::Engine::ants          include/aco/engine.hpp:84
 *   aco_gpu_get_best        <- Engine::best_length/best_tour engine.hpp:85-86
 *   aco_gpu_set_pheromone   <- (no reference equivalent: resynchronises tau, e.g.
 *                              for per-iteration atomic-path parity)
 *
 * Conventions (mirroring the reference):
 *  - No exceptions cross the boundary.  Every call returns aco_status; codes
 *    1..13 are 1 + (int)aco::Errc (errors.hpp:8-27) so a C++ wrapper can
 *    rethrow aco::Error{code}.  aco_gpu_last_error() has the message.
 *  - Host buffers are caller-owned and copied synchronously.
 *  - A context is single-owner and not thread-safe, like aco::Engine.
 *  - All matrices at the boundary are dense row-major n x n (Matrix<T>,
 *    matrix.hpp:12); the device uses padded pitches internally.
 *  - There is no CPU fallback: a context can only be created on a CUDA device.
 */
#ifndef ACO_GPU_H
#define ACO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ACO_OK = 0,
    /* 1 + aco::Errc (errors.hpp:8-27) */
    ACO_E_MISSING_FIELD = 1,
    ACO_E_UNSUPPORTED_EDGE_WEIGHT_TYPE = 2,
    ACO_E_MALFORMED_COORD = 3,
    ACO_E_DIMENSION_MISMATCH = 4,
    ACO_E_INDEX_OUT_OF_RANGE = 5,
    ACO_E_OVERFLOW = 6,
    ACO_E_INVALID_LENGTH = 7,
    ACO_E_NOT_A_PERMUTATION = 8,
    ACO_E_NOT_CLOSED = 9,
    ACO_E_ALL_VISITED = 10,
    ACO_E_INCONSISTENT_LENGTH = 11,
    ACO_E_IO_ERROR = 12,
    ACO_E_CONFIG_ERROR = 13,
    /* engine-side */
    ACO_E_CUDA = 100,
    ACO_E_NCCL = 101,
    ACO_E_UNSUPPORTED = 102
} aco_status;

/* aco::Selection (construction.hpp:13) */
enum { ACO_SEL_ROULETTE = 0, ACO_SEL_NN = 1, ACO_SEL_DATA_PARALLEL = 2 };
/* aco::Deposit (pheromone.hpp:16).  accumulate runs the atomic-scatter kernel
 * (red.global.add.f64); the three gather variants are bit-identical in the
 * reference (SURVEY [E2]) and all run the deterministic row-gather kernel. */
enum { ACO_DEP_ACCUMULATE = 0, ACO_DEP_SCATTER_GATHER = 1, ACO_DEP_SCATTER_GATHER_TILED = 2,
       ACO_DEP_SYMMETRIC_REDUCTION = 3 };
/* aco::EdgeWeightType (tsplib.hpp:16) */
enum { ACO_EUC_2D = 0, ACO_CEIL_2D = 1, ACO_ATT = 2 };
/* Construction weight stream. */
enum {
    ACO_STREAM_AUTO = 0, /* fp32 filter when it is exact-by-certification (default) */
    ACO_STREAM_FP64 = 1, /* fp64 rows, certified parallel scan + exact fallback */
    ACO_STREAM_FP32 = 2  /* fp32 row-scaled filter, fp64 certification + exact fallback */
};

/* aco::Parameters (model.hpp:29-53) + aco::RunConfig (engine.hpp:22-29). */
typedef struct {
    int32_t n;            /* cities (dist is n x n) */
    int32_t m;            /* ants; 0 means n (engine.hpp:60) */
    int32_t nn;           /* neighbour list length (nn selection) */
    int32_t theta;        /* tile size (data-parallel selection, ledger model) */
    int32_t selection;    /* ACO_SEL_* */
    int32_t deposit;      /* ACO_DEP_* */
    int32_t random_start; /* engine.hpp:104-111 */
    int32_t stream;       /* ACO_STREAM_* */
    double alpha, beta, rho;
    uint64_t seed;
    int32_t device;       /* CUDA device ordinal */
    /* Ant sharding: this context constructs global ants
     * [ant_begin, ant_end) of m; 0/0 means all.  With world > 1 the
     * per-iteration exchange runs over NCCL (nccl_id from rank 0, one id
     * per context).  world == 1 with a non-zero nccl_id runs the same
     * sharded protocol on a one-rank communicator. */
    int32_t rank, world;
    int32_t ant_begin, ant_end;
    uint8_t nccl_id[128];
    /* Accumulate-deposit arithmetic and (sharded) delta-tau exchange:
     *  ACO_WIRE_FP64 (default): fp64 reds; sharded: fp64 all-reduce of the
     *    local delta (ranks differ from a single-GPU colony only by the
     *    atomic order, ~1e-16);
     *  ACO_WIRE_FP32: sharded only, fp32 all-reduce (half the bytes, one
     *    2^-24 rounding per delta: tours after iteration 0 may depend on G);
     *  ACO_WIRE_FIXED64: every deposit as an exact int64 fixed-point sum
     *    (scale from the iteration's best length) — order-free, so tau is
     *    bit-identical run to run, on every rank and for every G; sharded:
     *    ncclUint64 all-reduce;
     *  ACO_WIRE_MULTIMEM: FIXED64 whose deposit reds go straight into an NVLS
     *    multicast object (every GPU's delta at once, multimem.red.add.u64)
     *    with a flag barrier through the same object: no collective (needs
     *    world > 1 on one NVSwitch node; world == 1 runs FIXED64, and so does
     *    a node where the multicast object cannot be created or its fabric
     *    handle exported — every rank agrees, aco_gpu_describe reports it).
     * Every rank of a colony must pass the same value. */
    int32_t wire;
    /* Debug mode (TourBuffer::make pheromone.hpp:67-90 and
     * tour_length model.hpp:205-220): every construction is followed by a
     * device check that each tour is closed, a permutation of 0..n-1 and of
     * the stored length; a violation fails the call with ACO_E_NOT_CLOSED /
     * ACO_E_NOT_A_PERMUTATION / ACO_E_INCONSISTENT_LENGTH.  Off by default. */
    int32_t validate_tours;
} aco_gpu_params;

enum { ACO_WIRE_FP64 = 0, ACO_WIRE_FP32 = 1, ACO_WIRE_FIXED64 = 2, ACO_WIRE_MULTIMEM = 3 };

/* aco::IterationRecord (engine.hpp:31-38) + device timings. */
typedef struct {
    int32_t iteration;     /* 1-based */
    int64_t best_length;   /* iteration best (all ants, all ranks) */
    double mean_length;
    double construct_ms;   /* construction + tour lengths + iteration stats */
    double update_ms;      /* exchange + evaporate + deposit + choice_info */
    double choice_ms;      /* part of update_ms spent in the choice pass (0 if fused) */
    double exchange_ms;    /* NCCL part of update_ms (0 at world == 1) */
    double construct_kernel_ms; /* the construction kernel alone */
    double ledger[4];      /* predicted_access_cost: global_loads, global_stores,
                              shared_loads, atomic_ops (pheromone.hpp:37-54, 366) */
    int64_t fallbacks;     /* construction steps resolved by the exact fallback walk
                              (roulette tier 3; nn: full-row argmax scans + exact folds) */
    int64_t best_so_far;   /* Engine::best_length after this iteration */
    int64_t certified_fp64; /* roulette steps the fp32 certification left open and the
                               fp64 re-sum over the staged row certified (tier 2) */
} aco_gpu_iter_record;

/* ---- host-side model (C++ in libaco_gpu.so; no device work) ---------- */
const char* aco_errc_name(int status);
/* parse TSPLIB NODE_COORD text: pass xs=ys=NULL to query *dimension. */
aco_status aco_parse_instance(const char* text, int32_t* dimension, int32_t* edge_weight_type,
                              double* xs, double* ys, int32_t capacity, char* name,
                              int32_t name_capacity);
aco_status aco_parse_tour(const char* text, int32_t* tour, int32_t capacity, int32_t* length);
aco_status aco_build_distances(int32_t n, const double* xs, const double* ys,
                               int32_t edge_weight_type, int32_t* dist);
aco_status aco_build_nn_lists(int32_t n, const int32_t* dist, int32_t nn, int32_t* out);
aco_status aco_greedy_tour_length(int32_t n, const int32_t* dist, int64_t* out);
aco_status aco_tour_length(int32_t n, const int32_t* dist, const int32_t* tour,
                           int32_t tour_len, int64_t* out);
aco_status aco_predicted_access_cost(int32_t deposit, int32_t n, int32_t m, int32_t theta,
                                     double out[4]);
/* Parameters::validate (model.hpp:39-53) with the engine's m = 0 -> n rule
 * applied by the caller; nn_selected as in the reference. */
aco_status aco_validate_parameters(double alpha, double beta, double rho, int32_t m, int32_t nn,
                                   int32_t iterations, int32_t tile_size, int32_t n,
                                   int32_t nn_selected);
/* RngStream::uniform_at (rng.hpp:74-80) on the host: the draw (seed;
 * iteration, ant, step, draw) — the same Philox4x32-10 the kernels run. */
double aco_uniform_at(uint64_t seed, uint32_t iteration, uint32_t ant, uint32_t step,
                      uint32_t draw);
const char* aco_last_error(void); /* last host-side error message (thread-local) */

/* ---- device engine --------------------------------------------------- */
typedef struct aco_gpu_ctx aco_gpu_ctx;

/* Validates (Parameters::validate), computes tau0 = m / C_greedy, the
 * eta^beta table (host libm pow, model.hpp:167), nn lists, uploads and
 * computes the initial choice_info — the Engine constructor. */
aco_status aco_gpu_create(const aco_gpu_params* params, const int32_t* dist,
                          aco_gpu_ctx** out);
void aco_gpu_destroy(aco_gpu_ctx* ctx);
const char* aco_gpu_last_error(const aco_gpu_ctx* ctx);

aco_status aco_gpu_set_pheromone(aco_gpu_ctx* ctx, const double* tau);
aco_status aco_gpu_compute_choice_info(aco_gpu_ctx* ctx);
/* Constructs this context's ants for the current iteration; fills the
 * construction half of the record (may be NULL). */
aco_status aco_gpu_construct(aco_gpu_ctx* ctx, aco_gpu_iter_record* rec);
/* Exchange (world > 1) + evaporate + deposit + choice_info + best-so-far,
 * advances the iteration counter. */
aco_status aco_gpu_update(aco_gpu_ctx* ctx, aco_gpu_iter_record* rec);
/* construct + update; optionally copies this context's tours (rows of n+1)
 * and lengths to host buffers. */
aco_status aco_gpu_iterate(aco_gpu_ctx* ctx, aco_gpu_iter_record* rec, int32_t* tours_out,
                           int64_t* lengths_out);

/* TourBuffer::make's validation (pheromone.hpp:67-90) of caller-supplied
 * closed tours (count rows of n+1 cities) and their stored lengths, on the
 * device: ACO_E_NOT_CLOSED / ACO_E_NOT_A_PERMUTATION /
 * ACO_E_INCONSISTENT_LENGTH for the first failing tour (ascending order). */
aco_status aco_gpu_validate_tours(aco_gpu_ctx* ctx, const int32_t* tours, const int64_t* lengths,
                                  int32_t count);
aco_status aco_gpu_get_pheromone(aco_gpu_ctx* ctx, double* tau);
aco_status aco_gpu_get_choice(aco_gpu_ctx* ctx, double* choice);
/* choice32 as the construction kernel streams it, de-permuted and unscaled
 * (diagnostic; ACO_E_UNSUPPORTED when the fp32 stream is off). */
aco_status aco_gpu_get_choice32(aco_gpu_ctx* ctx, float* choice, int32_t* row_scale_exp);
/* nn selection's per-row argmax cache (diagnostic): n x 128 city ids, the
 * row's best cities under (choice desc, index asc); -1 ends a short list,
 * entry 0 = -2 marks a row the construction always scans in full.
 * ACO_E_UNSUPPORTED when the cache is off (roulette, or ACO_NN_TOPK=0). */
aco_status aco_gpu_get_topk(aco_gpu_ctx* ctx, int32_t* topk, int32_t* k);
aco_status aco_gpu_get_tours(aco_gpu_ctx* ctx, int32_t* tours, int64_t* lengths);
aco_status aco_gpu_get_best(aco_gpu_ctx* ctx, int32_t* tour, int64_t* length);
/* Resolved configuration: m (after m=0 -> n), local ant range, tau0, stream. */
aco_status aco_gpu_get_info(aco_gpu_ctx* ctx, int32_t* m, int32_t* ant_begin, int32_t* ant_end,
                            double* tau0, int32_t* stream, int32_t* iteration);
/* The cudaStream_t (as void*) every kernel of this context runs on, so a
 * caller can time it with CUDA events on the launching stream. */
void* aco_gpu_stream(aco_gpu_ctx* ctx);
/* Exchange buffers of a sharded context (world > 1), device pointers:
 *   succ/pred [world][n][S] int32 (gather deposits), inv [world][S] fp64
 *   (1/C_k), delta n x P64 fp64 (accumulate).  With world > 1 and an all-zero
 *   nccl_id the context runs in EXTERNAL-EXCHANGE mode: aco_gpu_construct
 *   fills this rank's shard (and its local delta), the caller performs the
 *   all-gather / all-reduce itself, then calls aco_gpu_update.  (Used to test
 *   the sharded device path on one GPU; statistics are per shard.) */
aco_status aco_gpu_exchange_buffers(aco_gpu_ctx* ctx, void** succ, void** pred, void** inv,
                                    void** delta, int32_t* shard_stride, int32_t* P64);
/* Row-sharded gather deposit in EXTERNAL-EXCHANGE mode (world > 1, gather
 * deposit, rows of <= ~4000 doubles): after the caller delivered, from every
 * rank g, g's succ/pred rows [rank*B, rank*B + B) (B = ceil(n / world)) and
 * the 1/C_k blocks, folds this rank's row block into delta rows
 * [rank*B, rank*B + B) (delta row pitch P64); the caller then all-gathers the
 * delta row blocks and calls aco_gpu_update, which applies them to every row
 * (pheromone.hpp:213-228, bit-identical to the replicated fold).  With an
 * NCCL id the engine does this itself inside aco_gpu_update.  Without a
 * preceding aco_gpu_fold, aco_gpu_update folds all rows (replicated).
 * ACO_E_CONFIG_ERROR when the context does not row-shard; *row_blk = B. */
aco_status aco_gpu_fold(aco_gpu_ctx* ctx, int32_t* row_blk);
/* Human-readable name + launch shape of the last construction kernel
 * (e.g. "k_construct_roulette<float,19,1> grid=2392 per_sm=17 ..."); copies at
 * most len-1 bytes + NUL into buf, returns the full length.  Empty before the
 * first construction.  (No reference counterpart: diagnostics for bench.py.) */
int32_t aco_gpu_describe(const aco_gpu_ctx* ctx, char* buf, int32_t len);
/* Number of kernel launches issued by this context since creation. */
int64_t aco_gpu_launch_count(const aco_gpu_ctx* ctx);

/* NCCL unique id for world > 1 (rank 0 creates it, the caller distributes it). */
aco_status aco_gpu_nccl_unique_id(uint8_t out[128]);

/* The device replay of the host libm's pow (pow(tau, alpha) in choice_info
 * for alpha not in {0, 1}, model.hpp:167), for unit parity tests:
 * out[i] = pow(xs[i], ys[i]) for xs >= +0 finite, ys > 0 finite.
 * ACO_E_UNSUPPORTED when the host libm's pow tables cannot be located. */
aco_status aco_gpu_libm_pow(int32_t device, int32_t count, const double* xs, const double* ys,
                            double* out);

/* Device self-test helpers (unit parity of the device RNG / scan pieces). */
aco_status aco_gpu_philox_uniform(int32_t device, uint64_t seed, uint32_t iteration,
                                  uint32_t ant, int32_t count, const uint32_t* steps,
                                  const uint32_t* draws, double* out);

#ifdef __cplusplus
}
#endif
#endif /* ACO_GPU_H */
