// libaco_gpu.so — C-ABI implementation (include/aco_gpu.h).
//
// One context = one GPU = one colony shard.  All iteration state (tau,
// choice, tours, lengths, best tour) stays resident in HBM/L2; the host only
// sees what the caller asks for.  Multi-GPU sharding uses NCCL,
// loaded at run time with dlopen so a single-GPU process never needs it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/aco_gpu.h"
#include "construct.cuh"
#include "host_model.hpp"
#include "update.cuh"

using namespace acob200;

// ---------------------------------------------------------------------------
// NCCL, resolved lazily.
namespace {

struct NcclApi {
    bool loaded = false;
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.loaded) {
        api.loaded = true;
        // ACO_NCCL_LIB: load another NCCL-compatible library instead (the
        // tests' in-process loopback, tests/loopnccl, which runs several ranks
        // on one GPU — real NCCL refuses that)
        if (const char* lib = std::getenv("ACO_NCCL_LIB")) api.handle = dlopen(lib, RTLD_NOW | RTLD_LOCAL);
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            if (api.handle) break;
            api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        }
        if (api.handle) {
            auto sym = [&](const char* s) { return dlsym(api.handle, s); };
            api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
            api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
            api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
            api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
            api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
            api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
            api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
            api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
            api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
            api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
            api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        }
    }
    return api;
}

// CUDA driver entry points for the NVLS multicast exchange (f2), resolved
// through the runtime so libaco_gpu.so never links libcuda directly.
struct DriverApi {
    bool loaded = false;
    CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                                 unsigned long long) = nullptr;
    CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                           unsigned long long) = nullptr;
    CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
    CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*GetErrorName)(CUresult, const char**) = nullptr;
};

DriverApi& driver() {
    static DriverApi d;
    if (!d.loaded) {
        d.loaded = true;
        auto get = [](const char* name, auto& fn) {
            void* p = nullptr;
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
            cudaGetLastError();
        };
        get("cuMulticastGetGranularity", d.MulticastGetGranularity);
        get("cuMulticastCreate", d.MulticastCreate);
        get("cuMulticastAddDevice", d.MulticastAddDevice);
        get("cuMulticastBindMem", d.MulticastBindMem);
        get("cuMulticastUnbind", d.MulticastUnbind);
        get("cuMemCreate", d.MemCreate);
        get("cuMemRelease", d.MemRelease);
        get("cuMemExportToShareableHandle", d.MemExportToShareableHandle);
        get("cuMemImportFromShareableHandle", d.MemImportFromShareableHandle);
        get("cuMemAddressReserve", d.MemAddressReserve);
        get("cuMemAddressFree", d.MemAddressFree);
        get("cuMemMap", d.MemMap);
        get("cuMemUnmap", d.MemUnmap);
        get("cuMemSetAccess", d.MemSetAccess);
        get("cuGetErrorName", d.GetErrorName);
    }
    return d;
}

thread_local std::string g_host_err;

struct Fail {
    aco_status code;
    std::string msg;
};

} // namespace

// ---------------------------------------------------------------------------
struct aco_gpu_ctx {
    // configuration
    Config cfg;
    int n = 0, m = 0, stream_kind = ACO_STREAM_FP32;
    uint64_t seed = 1;
    int random_start = 0;
    int rank = 0, world = 1, ant_begin = 0, ant_end = 0, mloc = 0, S = 0;
    int P64 = 0, PW = 0, NV = 0, V = 4, C = 0, R = 1, MAXR = 1, tabu_words = 0;
    int LA = 32;          // lanes sharing a streamed row
    bool nat = false;     // streamed rows in the natural layout (RowLayout; plain launches, odd NV)
    bool exact_only = false; // k_construct_roulette_exact (rows too long to stream)
    int32_t* host_tours = nullptr; // this construction's streamed host tour buffer (device view)
    double tau0 = 0.0;
    int64_t max_d = 0;
    int device = 0, num_sms = 0;
    int construct_grid = 0;
    std::string construct_desc;  // kernel + launch shape of the last construction
    bool fused_tail = false;     // the last construction kernel also formed len/inv(/succ/pred)
    int iteration = 0;
    int64_t best_so_far = std::numeric_limits<int64_t>::max();
    int64_t launches = 0;
    std::string err;

    // device buffers
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr; // D2H of the tours, overlapped with the update
    cudaEvent_t ev[6] = {};
    int32_t* d_dist = nullptr;
    double* d_lut = nullptr;
    double* d_etab = nullptr;
    double* d_tau = nullptr;
    double* d_choice = nullptr;
    float* d_choice32 = nullptr;
    double* d_choice_p64 = nullptr;
    int32_t* d_scale = nullptr;
    int32_t* d_nn = nullptr;
    double* d_choice_nn = nullptr; // n x nn
    int2* d_choice_nn32 = nullptr;  // n x nn {id, row-scaled fp32 weight bits} (nn <= 32)
    int32_t* d_nn_scale = nullptr;  // n
    int32_t* d_topk = nullptr;     // n x kTopK argmax cache (nn selection)
    long long last_fb[2] = {0, 0}; // last construction: exact/full-scan, argmax fallbacks
    int32_t* d_tours = nullptr;
    int64_t* d_len = nullptr;
    double* d_inv = nullptr;   // [world][S]
    int32_t* d_succ = nullptr; // [world][n][S]
    int32_t* d_pred = nullptr;
    double* d_delta = nullptr;
    bool sym = false; // one-GPU accumulate: symmetric upper-triangle delta (k_deposit_sym)
    float* d_delta32 = nullptr; // sharded atomic path over NCCL: the fp32 wire copy of d_delta
    long long* d_stats = nullptr;   // [0..2] stats, [3] best_so_far
    int32_t* d_best = nullptr;      // n+1
    unsigned long long* d_fb = nullptr; // [0] exact fallbacks, [1] nn argmax fallbacks, [2] roulette tier-2
    unsigned long long* d_timing = nullptr; // ACO_TIMING phase cycles
    long long* h_stats = nullptr;       // pinned: [0..7] d_stats, [8..9] fallback counters
    int32_t* d_tourbuf = nullptr;       // sharded: winning tour exchange buffer (n+1)
    LibmPowTables* d_powtab = nullptr;  // alpha not in {0, 1}: the host libm's pow tables
    // fixed-point accumulate (wire FIXED64 / MULTIMEM): exact int64 delta sums
    bool fixed = false;
    bool multimem = false;              // NVLS multicast exchange (world > 1)
    unsigned long long* d_delta_fix = nullptr; // n x P64 (or the multicast object's local memory)
    // NVLS multicast object (f2): delta + barrier flag, local (uc) and multicast (mc) views
    CUmemGenericAllocationHandle mc_handle = 0, mc_phys = 0;
    CUdeviceptr mc_uc = 0, mc_va = 0;
    size_t mc_size = 0;
    unsigned long long mc_epoch = 0;
    bool mc_fallback = false; // MULTIMEM requested, multicast unavailable: FIXED64 all-reduce
    // nn + fixed-point accumulate: compact int64 slots + non-list edge records
    unsigned long long* d_dnn_fix = nullptr;   // n x nn
    DepositRecord* d_rec = nullptr;            // this rank's records (capacity mloc * n)
    DepositRecord* d_rec_all = nullptr;        // [world][rec_stride] after the all-gather
    size_t rec_stride = 0;                     // records per rank in d_rec_all
    unsigned long long* d_rec_counts = nullptr; // [world]: gathered counts ([rank] = own)
    unsigned long long* h_rec_counts = nullptr; // pinned copy
    uint8_t* d_qpos = nullptr;          // nn + accumulate: list position of every step's choice
    // roulette relay (leftover ants built in segments by several warps)
    unsigned long long* d_relay_flag = nullptr; // [num_sms]
    int32_t* d_relay_cur = nullptr;             // [num_sms]
    uint32_t* d_relay_tabu = nullptr;           // [num_sms][tabu_words]
    unsigned long long relay_epoch = 0;
    // resolved roulette launch shape, [0] plain / [1] streaming tours to host
    struct RouletteLaunch {
        bool valid = false, relay = false;
        void (*fn)(acob200::ConstructParams) = nullptr;
        size_t smem = 0;
        int grid = 0, W = 0, E = 0, K = 0;
        std::string desc;
    } rlaunch[2];
    double* d_dnn = nullptr;            // nn + accumulate: compact n x nn deposit slots
    // gather deposit with world > 1: row-sharded fold (rank r folds rows
    // [r*row_blk, (r+1)*row_blk) into delta rows, which are all-gathered)
    bool row_shard = false;
    int row_blk = 0;
    bool folded = false; // external mode: aco_gpu_fold ran this iteration
    ncclComm_t comm = nullptr;
    bool external = false; // world > 1 without an NCCL id: the caller exchanges
    bool sharded = false;  // the sharded protocol (world > 1, or a 1-rank NCCL communicator)
    int key_shift = 24;         // sharded iteration-best key: (length << key_shift) | ant
    bool key_two_stage = false; // lengths too long to pack: MIN length, then MIN ant
    bool validate_tours = false;      // debug mode: k_validate_tours after every construction
    unsigned long long* d_verr = nullptr;
};

namespace {

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw Fail{ACO_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};  \
    } while (0)

#define NK(call)                                                                         \
    do {                                                                                 \
        ncclResult_t r_ = (call);                                                        \
        if (r_ != ncclSuccess)                                                           \
            throw Fail{ACO_E_NCCL, std::string(#call) + ": " +                           \
                                       (nccl().GetErrorString ? nccl().GetErrorString(r_) \
                                                              : "nccl error")};          \
    } while (0)

template <class F>
aco_status guard_ctx(aco_gpu_ctx* ctx, F&& f) {
    try {
        f();
        return ACO_OK;
    } catch (const Fail& e) {
        if (ctx) ctx->err = e.msg;
        g_host_err = e.msg;
        return e.code;
    } catch (const ModelError& e) {
        if (ctx) ctx->err = e.what();
        g_host_err = e.what();
        return static_cast<aco_status>(1 + static_cast<int>(e.code));
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        g_host_err = e.what();
        return ACO_E_CUDA;
    }
}

void check_launch(aco_gpu_ctx* c, const char* what) {
    ++c->launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Fail{ACO_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

int round_up(int x, int a) { return (x + a - 1) / a * a; }

// ACO_DEBUG=1 prints each construction launch shape (read once per process)
bool debug_enabled() {
    static const bool on = std::getenv("ACO_DEBUG") != nullptr;
    return on;
}

__global__ void k_fill(double* p, size_t count, double v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

// ---- construction kernel dispatch ------------------------------------------
using ConstructFn = void (*)(ConstructParams);

// the relay variant (fp32 stream, single-round rows only)
template <bool ST, bool HI>
ConstructFn pick_roulette_relay_h(int NV) {
    switch (NV) {
    case 2: return k_construct_roulette_relay<2, ST, HI>;
    case 4: return k_construct_roulette_relay<4, ST, HI>;
    case 8: return k_construct_roulette_relay<8, ST, HI>;
    case 12: return k_construct_roulette_relay<12, ST, HI>;
    case 16: return k_construct_roulette_relay<16, ST, HI>;
    case 19: return k_construct_roulette_relay<19, ST, HI>;
    default: return k_construct_roulette_relay<20, ST, HI>;
    }
}
template <bool ST>
ConstructFn pick_roulette_relay(int NV, bool hi) {
    return hi ? pick_roulette_relay_h<ST, true>(NV) : pick_roulette_relay_h<ST, false>(NV);
}

template <typename WT, bool ST, bool HI>
ConstructFn pick_roulette_h(int NV, int MAXR, bool nat) {
    if (MAXR == 1) {
        switch (NV) {
        case 2: return k_construct_roulette<WT, 2, 1, ST, HI>;
        case 4: return k_construct_roulette<WT, 4, 1, ST, HI>;
        case 8: return k_construct_roulette<WT, 8, 1, ST, HI>;
        case 12: return k_construct_roulette<WT, 12, 1, ST, HI>;
        case 16: return k_construct_roulette<WT, 16, 1, ST, HI>;
        case 19:
            if constexpr (sizeof(WT) == 4)
                if (nat) return k_construct_roulette<WT, 19, 1, ST, HI, true>;
            return k_construct_roulette<WT, 19, 1, ST, HI>;
        default: return k_construct_roulette<WT, 20, 1, ST, HI>;
        }
    }
    return k_construct_roulette<WT, 20, 8, ST>;
}
// hi: a high-occupancy launch (>= kHiWarps warps per SM): the issue-lean step
// (in-place scans, predicated sequential group sums), fp32 stream only;
// nat: the natural row layout (odd NV)
template <typename WT, bool ST>
ConstructFn pick_roulette_s(int NV, int MAXR, bool hi, bool nat) {
    if constexpr (sizeof(WT) == 4)
        if (hi) return pick_roulette_h<WT, ST, true>(NV, MAXR, nat);
    return pick_roulette_h<WT, ST, false>(NV, MAXR, nat);
}
// stream = true: the variant that also streams tours into mapped host memory
template <typename WT>
ConstructFn pick_roulette(int NV, int MAXR, bool stream = false, bool hi = false, bool nat = false) {
    return stream ? pick_roulette_s<WT, true>(NV, MAXR, hi, nat) : pick_roulette_s<WT, false>(NV, MAXR, hi, nat);
}

int relay_min_q();
// Will the roulette construction use the relay launch (see the launch
// below)?  Decides the streamed-row layout before the first launch; the
// launch never relays a natural-layout context.
bool relay_predicted(const aco_gpu_ctx* c) {
    if (c->num_sms <= 0 || c->mloc <= 0) return false;
    const int q = c->mloc / c->num_sms, E = c->mloc - q * c->num_sms;
    return E > 0 && q >= relay_min_q() && q % 4 == 0 && q * c->num_sms >= 32 * E;
}

void choose_stream_layout(aco_gpu_ctx* c) {
    c->V = (c->stream_kind == ACO_STREAM_FP64) ? 2 : 4;
    c->LA = 32;
    static const int nvs[] = {2, 4, 8, 12, 16, 19, 20};
    c->NV = 0;
    for (int nv : nvs)
        if (32 * nv * c->V >= c->n) {
            c->NV = nv;
            break;
        }
    if (c->NV) {
        c->MAXR = 1;
        c->R = 1;
    } else {
        c->NV = 20;
        c->MAXR = 8;
        c->R = (c->n + 32 * 20 * c->V - 1) / (32 * 20 * c->V);
    }
    const char* ex = std::getenv("ACO_ROULETTE_EXACT");
    if (c->cfg.selection == ACO_SEL_ROULETTE && (c->R > 8 || (ex && ex[0] == '1'))) {
        // rows too long for the streamed layouts: exact replay every step
        c->exact_only = true;
        c->NV = 20;
        c->MAXR = 8;
        c->R = 1;
        c->C = c->NV * c->V;
        c->PW = 0;
        c->tabu_words = (c->n + 31) / 32 + 2;
        return;
    }
    c->C = c->NV * c->V;
    // physical row length: the natural layout (odd NV) when the launch will
    // be the plain one-warp-per-ant kernel, else with pad slots
    c->nat = (c->NV & 1) && c->MAXR == 1 && c->stream_kind == ACO_STREAM_FP32 && !relay_predicted(c);
    c->PW = c->R * (c->nat ? 32 : kLP) * c->C;
    c->tabu_words = c->R * c->C + 4;  // covers R*32*C cities; even, keeps the fp64 area 8-aligned
}

// nn selection: rebuild the per-row argmax cache after every choice update
void launch_topk(aco_gpu_ctx* c) {
    if (!c->d_topk) return;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_row_topk, kTopThreads, 0));
    const int grid = std::max(1, std::min(c->n, std::max(1, per_sm) * c->num_sms));
    k_row_topk<<<grid, kTopThreads, 0, c->stream>>>(c->d_choice, c->n, c->P64, c->d_topk);
    check_launch(c, "k_row_topk");
}

// host-side launch modes of the row-sharded gather (c->row_shard): fold this
// rank's row block into delta rows / apply the (all-gathered) delta rows
constexpr int MODE_FOLD_OWN = 100, MODE_APPLY = 101;

void launch_rows(aco_gpu_ctx* c, int mode) {
    RowParams rp{};
    rp.tau = c->d_tau;
    rp.choice64 = c->d_choice;
    rp.choice32 = c->d_choice32;
    rp.choice_perm64 = c->d_choice_p64;
    rp.scale_exp = c->d_scale;
    rp.dist = c->d_dist;
    rp.lut = c->d_lut;
    rp.etab = c->d_etab;
    rp.delta = c->d_delta;
    rp.delta32 = c->d_delta32;
    rp.succ = c->d_succ;
    rp.pred = c->d_pred;
    rp.inv = c->d_inv;
    rp.nn_lists = c->d_nn;
    rp.choice_nn = c->d_choice_nn;
    rp.choice_nn32 = c->d_choice_nn32;
    rp.nn_scale = c->d_nn_scale;
    rp.nn = c->cfg.nn;
    rp.n = c->n;
    rp.P64 = c->P64;
    rp.PW = c->PW;
    rp.C = c->C;
    rp.V = c->V;
    rp.LA = c->LA;
    rp.nat = c->nat ? 1 : 0;
    rp.shards = c->world;
    rp.S = c->S;
    rp.m = !c->sharded ? c->mloc : c->m; // a local ant range is one shard of mloc ants
    rp.alpha = c->cfg.alpha;
    rp.keep = 1.0 - c->cfg.rho; // pheromone.hpp:179
    rp.powtab = c->d_powtab;
    rp.delta_fix = c->d_delta_fix;
    rp.stats = c->d_stats;
    rp.row_begin = 0;
    rp.row_end = c->n;
    if (mode == MODE_FOLD_OWN || mode == MODE_APPLY) { // row-sharded gather (c->row_shard)
        if (mode == MODE_FOLD_OWN) {
            rp.row_begin = std::min(c->n, c->rank * c->row_blk);
            rp.row_end = std::min(c->n, rp.row_begin + c->row_blk);
            const size_t wsmem0 = static_cast<size_t>(c->P64) * sizeof(double) + 64 * sizeof(double);
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows_gather_warp<false>, 32, wsmem0));
            const int grid = std::max(1, std::min(std::max(1, rp.row_end - rp.row_begin), per_sm * c->num_sms));
            k_rows_gather_warp<false><<<grid, 32, wsmem0, c->stream>>>(rp);
            check_launch(c, "k_rows_gather_warp");
            return;
        }
        const size_t dsmem = (rp.choice32 || rp.choice_perm64) ? static_cast<size_t>(c->P64) * sizeof(double) : 0;
        if (dsmem > 48 * 1024)
            CK(cudaFuncSetAttribute(k_rows<MODE_DELTA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
        k_rows<MODE_DELTA><<<std::min(c->n, c->num_sms * 8), 256, dsmem, c->stream>>>(rp);
        check_launch(c, "k_rows");
        launch_topk(c);
        return;
    }
    const size_t smem = static_cast<size_t>(c->P64) * sizeof(double);
    const size_t wsmem = smem + 64 * sizeof(double);
    if (mode == MODE_GATHER && wsmem <= 32 * 1024) { // one warp per row
        // Default: fold-only warp kernel (ordered sums -> delta rows) and the
        // tau/choice epilogue by k_rows<DELTA> at full CTA occupancy (pr2392:
        // 0.26 -> 0.20 ms); ACO_GATHER_SPLIT=0 keeps the epilogue in the warp
        // kernel.
        const bool split = c->d_delta != nullptr;
        auto fn = split ? k_rows_gather_warp<false> : k_rows_gather_warp<true>;
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32, wsmem));
        const int grid = std::max(1, std::min(c->n, per_sm * c->num_sms));
        fn<<<grid, 32, wsmem, c->stream>>>(rp);
        check_launch(c, "k_rows_gather_warp");
        if (split) {
            const size_t dsmem = (rp.choice32 || rp.choice_perm64) ? smem : 0;
            if (dsmem > 48 * 1024)
                CK(cudaFuncSetAttribute(k_rows<MODE_DELTA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)dsmem));
            k_rows<MODE_DELTA><<<std::min(c->n, c->num_sms * 8), 256, dsmem, c->stream>>>(rp);
            check_launch(c, "k_rows");
        }
        launch_topk(c);
        return;
    }
    // the CTA kernel needs the shared row only for the gather fold and the
    // permuted streamed copies (k_rows)
    const bool use_row = mode == MODE_GATHER || rp.choice32 || rp.choice_perm64;
    const size_t rsmem = use_row ? smem : 0;
    const int grid = std::min(c->n, c->num_sms * 8);
    if (smem > 48 * 1024) {
        CK(cudaFuncSetAttribute(k_rows<MODE_CHOICE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_rows<MODE_GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_rows<MODE_DELTA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_rows<MODE_DELTA32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_rows<MODE_DELTA_FIX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_rows<MODE_DELTA_SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    if (mode == MODE_CHOICE) k_rows<MODE_CHOICE><<<grid, 256, rsmem, c->stream>>>(rp);
    else if (mode == MODE_GATHER) k_rows<MODE_GATHER><<<grid, 256, rsmem, c->stream>>>(rp);
    else if (mode == MODE_DELTA32) k_rows<MODE_DELTA32><<<grid, 256, rsmem, c->stream>>>(rp);
    else if (mode == MODE_DELTA_FIX) k_rows<MODE_DELTA_FIX><<<grid, 256, rsmem, c->stream>>>(rp);
    else if (mode == MODE_DELTA_SYM) k_rows<MODE_DELTA_SYM><<<grid, 256, rsmem, c->stream>>>(rp);
    else k_rows<MODE_DELTA><<<grid, 256, rsmem, c->stream>>>(rp);
    check_launch(c, "k_rows");
    launch_topk(c);
}

bool gather_mode(const aco_gpu_ctx* c) { return c->cfg.deposit != ACO_DEP_ACCUMULATE; }

// directed float roundings of a double (the host twins of __double2float_ru/rd)
float f32_ru(double x) {
    float f = static_cast<float>(x);
    if (static_cast<double>(f) < x) f = std::nextafter(f, std::numeric_limits<float>::infinity());
    return f;
}
float f32_rd(double x) {
    float f = static_cast<float>(x);
    if (static_cast<double>(f) > x) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
    return f;
}

// nn fast-path certification constants (k_construct_nn): e counts the fp32
// quantisation (1 ulp), 5 scan levels, margins and the reference's nn
// sequential fp64 adds; nn * 2^-149 bounds the subnormal losses; rounded
// outward so the fp32 compares imply the exact ones
void nn_certify_constants(ConstructParams& p, int nn) {
    const double nn_e = (12.0 * 0x1.0p-24 + static_cast<double>(nn + 8) * 0x1.0p-53) * (1.0 + 0x1.0p-16);
    p.nn_e32 = f32_ru(nn_e);
    p.nn_lo32 = f32_rd(1.0 - nn_e);
    p.nn_ce = f32_ru(nn_e + 4.0 * 0x1.0p-24);
    p.nn_absq = static_cast<float>(nn) * 0x1.0p-149f; // exact: a subnormal multiple
}

ConstructParams make_cp(aco_gpu_ctx* c) {
    ConstructParams p{};
    p.w = c->stream_kind == ACO_STREAM_FP64 ? static_cast<const void*>(c->d_choice_p64)
                                            : static_cast<const void*>(c->d_choice32);
    p.w64 = c->d_choice;
    p.nn_lists = c->d_nn;
    p.choice_nn = c->d_choice_nn;
    p.choice_nn32 = c->d_choice_nn32;
    p.tours = c->d_tours;
    p.fallbacks = c->d_fb;
    p.argmax_fallbacks = c->d_fb + 1;
    p.tier2 = c->d_fb + 2;
    p.n = c->n;
    p.P64 = c->P64;
    p.PW = c->PW;
    p.R = c->R;
    p.nn = c->cfg.nn;
    p.ant_begin = c->ant_begin;
    p.mloc = c->mloc;
    p.random_start = c->random_start;
    p.theta = c->cfg.theta;
    p.tabu_words = c->tabu_words;
    p.iteration = static_cast<uint32_t>(c->iteration);
    p.seed = c->seed;
    p.timing = c->d_timing;
    p.topk = c->d_topk;
    p.topk_k = kTopK;
    p.host_tours = c->host_tours;
    p.dist = c->d_dist;
    p.inv_out = c->d_inv + static_cast<size_t>(c->rank) * c->S;
    if (gather_mode(c)) {
        p.succ_out = c->d_succ + static_cast<size_t>(c->rank) * c->n * c->S;
        p.pred_out = c->d_pred + static_cast<size_t>(c->rank) * c->n * c->S;
    }
    p.S = c->S;
    p.qpos = c->d_qpos;
    nn_certify_constants(p, c->cfg.nn);
    return p;
}

// roulette relay: minimum warps per SM (ACO_RELAY=0 disables, ACO_RELAY=q
// sets the threshold) and the segment count override (ACO_RELAY_K)
int relay_min_q() {
    static const int q = [] {
        const char* e = std::getenv("ACO_RELAY");
        return e ? (std::atoi(e) <= 0 ? 1 << 30 : std::atoi(e)) : 8;
    }();
    return q;
}
int relay_k_override() {
    static const int k = [] {
        const char* e = std::getenv("ACO_RELAY_K");
        return e ? std::atoi(e) : 0;
    }();
    return k;
}

// the nn kernel forms the tour lengths in its tail (tour_tail);
// ACO_FUSED_TAIL=0 keeps the separate k_tour_length launch
bool fused_tail_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ACO_FUSED_TAIL");
        return ACO_FUSED_TAIL_BUILD && !(e && e[0] == '0');
    }();
    return on;
}

void launch_construct(aco_gpu_ctx* c) {
    ConstructParams p = make_cp(c);
    c->fused_tail = false;
    const size_t smem1 = static_cast<size_t>(c->tabu_words) * sizeof(uint32_t);
    if (c->mloc == 0) return;
    if (c->cfg.selection == ACO_SEL_ROULETTE && c->exact_only) {
        const uint32_t stage_bytes = 16 * 1024;
        const size_t smem = 128 + stage_bytes + smem1 + static_cast<size_t>((c->n + 31) / 32) * sizeof(double) + 8;
        if (smem > 48 * 1024)
            CK(cudaFuncSetAttribute(k_construct_roulette_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_construct_roulette_exact, 32, smem));
        const int grid = std::max(1, std::min(c->mloc, std::max(1, per_sm) * c->num_sms));
        c->construct_grid = grid;
        c->construct_desc = "k_construct_roulette_exact grid=" + std::to_string(grid);
        k_construct_roulette_exact<<<grid, 32, smem, c->stream>>>(p, stage_bytes);
        check_launch(c, "k_construct_roulette_exact");
    } else if (c->cfg.selection == ACO_SEL_ROULETTE) {
        const bool st = c->host_tours != nullptr;
        // the launch shape (kernel, shared memory, grid, relay split) is
        // resolved once per context and tours-to-host mode: the occupancy
        // queries and attribute calls stay off the per-iteration host path,
        // where the GPU would idle waiting for the first launch
        auto& L = c->rlaunch[st ? 1 : 0];
        if (!L.valid) {
        // the warps each SM will hold: >= kHiWarps -> the issue-lean step
        constexpr int kHiWarps = 12;
        const bool hi = (c->mloc + c->num_sms - 1) / c->num_sms >= kHiWarps;
        ConstructFn fn = c->stream_kind == ACO_STREAM_FP64 ? pick_roulette<double>(c->NV, c->MAXR, st)
                                                           : pick_roulette<float>(c->NV, c->MAXR, st, hi, c->nat);
        const size_t wsz = c->stream_kind == ACO_STREAM_FP64 ? sizeof(double) : sizeof(float);
        const int ng = (c->NV + 3) / 4;
        size_t smem = 128 + static_cast<size_t>(c->PW) * wsz + smem1 +
                            static_cast<size_t>((c->n + 31) / 32) * sizeof(double) +
                            (c->MAXR > 1 ? static_cast<size_t>(c->MAXR) * ng * 32 * wsz : 0);
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32, smem));
        int grid = std::max(1, std::min(c->mloc, per_sm * c->num_sms));
        // Relay: with q = floor(mloc / SMs) >= relay_min_q warps on every SM
        // and E = mloc - q*SMs leftover ants, one warp per SM-slot builds its
        // own ant and the E leftovers are built in K segments by K different
        // warps each (handing over through global memory), instead of E SMs
        // running a (q+1)-th warp for the whole kernel: that warp shares an SM
        // sub-partition (5 warps on one scheduler at q = 16) and is the last to
        // finish — at pr2392 ONE leftover ant costs 9.5% (m = 2368: 3.68 ms,
        // m = 2369: 4.02 ms); relayed, m = 2392 (16 x 148 + 24) runs 3.78 ms
        // instead of 4.12 (tools/relay_ab.py, same tours).
        const int q = c->mloc / c->num_sms;
        const int E = c->mloc - q * c->num_sms;
        std::string relay_desc;
        // Only when the leftovers are few (W >= 32 E: every relay warp carries
        // at most ~1/32 of an ant more); pr1002 (E = 114 of 888) runs slower
        // relayed (0.82 -> 1.03 ms, tools/relay_ab.py).
        // The leftover warp only hurts where it creates a new busiest SM
        // sub-partition (a one-warp CTA lands on one of 4 schedulers): q a
        // multiple of 4.  Measured (profiles/relay_q_ab_r02.txt): relay wins
        // at q = 8 (-4.6%) and 16 (-8%), loses at q = 4 (+2.7%) and 5-7 (+6-7%).
        if (c->stream_kind == ACO_STREAM_FP32 && c->MAXR == 1 && E > 0 && q >= relay_min_q() &&
            q % 4 == 0 && q <= per_sm && q * c->num_sms >= 32 * E && !c->nat) {
            ConstructFn rfn = st ? pick_roulette_relay<true>(c->NV, hi) : pick_roulette_relay<false>(c->NV, hi);
            const size_t rsmem = smem + smem1;
            CK(cudaFuncSetAttribute(rfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rsmem)));
            int rper_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rper_sm, rfn, 32, rsmem));
            const int W = q * c->num_sms;
            // K ~ sqrt(n) segments of >= 64 steps (pr2392: K = 37; 20 and 49-74
            // measured no better, profiles/relay_k_ab_r02.txt)
            int K = relay_k_override();
            if (K <= 0)
                K = std::min(static_cast<int>(std::lround(std::sqrt(static_cast<double>(c->n - 1)))),
                             (c->n - 1) / 64);
            K = std::max(1, std::min({K, W / E, (c->n - 1) / 33}));
            if (rper_sm >= q && K >= 1 && (c->n - 1) / K >= 33) {
                if (!c->d_relay_flag) {
                    CK(cudaMalloc(&c->d_relay_flag, c->num_sms * sizeof(unsigned long long)));
                    CK(cudaMemsetAsync(c->d_relay_flag, 0, c->num_sms * sizeof(unsigned long long), c->stream));
                    CK(cudaMalloc(&c->d_relay_cur, c->num_sms * sizeof(int32_t)));
                    CK(cudaMalloc(&c->d_relay_tabu,
                                  static_cast<size_t>(c->num_sms) * c->tabu_words * sizeof(uint32_t)));
                }
                L.relay = true;
                L.W = W;
                L.E = E;
                L.K = K;
                fn = rfn;
                smem = rsmem;
                per_sm = rper_sm;
                grid = W;
                relay_desc = " relay: W=" + std::to_string(W) + " E=" + std::to_string(E) +
                             " K=" + std::to_string(K);
            }
        }
        L.fn = fn;
        L.smem = smem;
        L.grid = grid;
        L.desc = std::string("k_construct_roulette<") +
                 (c->stream_kind == ACO_STREAM_FP64 ? "double," : "float,") +
                 std::to_string(c->NV) + "," + std::to_string(c->MAXR) + (hi ? ",hi" : "") + (c->nat ? ",nat" : "") + "> grid=" +
                 std::to_string(grid) + " per_sm=" + std::to_string(per_sm) +
                 " smem=" + std::to_string(smem) + " row=" + std::to_string(c->PW) +
                 (st ? " streams_tours_to_host" : "") + relay_desc;
        L.valid = true;
        }
        if (L.relay) {
            // fused tour tail only at high occupancy, where it overlaps other
            // warps' steps (m = n = 2392: construct 3.853 -> 3.834 ms); with
            // 4-8 warps per SM it lengthens the kernel more than the
            // k_tour_length launch it saves (1196 ants: 2.820 -> 2.874 ms)
            if (fused_tail_enabled() && L.W >= 12 * c->num_sms) {
                p.len_out = c->d_len;
                c->fused_tail = true;
            }
            p.relay_W = L.W;
            p.relay_E = L.E;
            p.relay_K = L.K;
            p.relay_epoch = ++c->relay_epoch;
            p.relay_flag = c->d_relay_flag;
            p.relay_cur = c->d_relay_cur;
            p.relay_tabu = c->d_relay_tabu;
        }
        c->construct_grid = L.grid;
        c->construct_desc = L.desc;
        if (debug_enabled())
            std::fprintf(stderr, "construct: %s\n", c->construct_desc.c_str());
        L.fn<<<L.grid, 32, L.smem, c->stream>>>(p);
        check_launch(c, "k_construct_roulette");
    } else if (c->cfg.selection == ACO_SEL_NN) {
        // Early request of the crossing candidate's list (before its
        // certification, k_construct_nn<true>, 64 registers) pays when the
        // launch is latency-bound — few ants per SM: 10k with 1250 ants 8.06
        // -> 7.56 ms, pr1002 0.678 -> 0.649 ms — and costs at full occupancy
        // (10k, 10000 ants: 27.5 -> 30.6 ms; tools/lib_ab.py).
        // ACO_NN_SPEC=0/1 forces the choice.
        static const int spec_env = [] {
            const char* e = std::getenv("ACO_NN_SPEC");
            return e ? (e[0] == '1' ? 1 : 0) : -1;
        }();
        const bool spec = spec_env >= 0 ? spec_env == 1 : c->mloc <= 12 * c->num_sms;
        const bool f32 = c->cfg.nn <= 32 && c->d_choice_nn32 != nullptr;
        auto nnfn = f32 ? (spec ? k_construct_nn<true, true> : k_construct_nn<false, true>)
                        : (spec ? k_construct_nn<true, false> : k_construct_nn<false, false>);
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nnfn, 32, smem1));
        const int grid = std::max(1, std::min(c->mloc, per_sm * c->num_sms));
        c->construct_grid = grid;
        c->construct_desc = "k_construct_nn grid=" + std::to_string(grid) +
                            " per_sm=" + std::to_string(per_sm) + (spec ? " spec" : "");
        if (fused_tail_enabled()) {
            p.len_out = c->d_len;
            c->fused_tail = true;
        }
        nnfn<<<grid, 32, smem1, c->stream>>>(p);
        check_launch(c, "k_construct_nn");
    } else {
        const size_t smem4 = smem1 * 4 + 4 * 1024 * sizeof(int);
        if (smem4 > 48 * 1024)
            CK(cudaFuncSetAttribute(k_construct_data_parallel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4));
        const int grid = std::max(1, (c->mloc + 3) / 4);
        c->construct_grid = grid;
        c->construct_desc = "k_construct_data_parallel grid=" + std::to_string(grid);
        k_construct_data_parallel<<<grid, 128, smem4, c->stream>>>(p);
        check_launch(c, "k_construct_data_parallel");
    }
}


// ---- NVLS multicast object for the fused exchange (wire MULTIMEM, f2) -----
// Rank 0 creates a multicast object over `world` devices and exports it as a
// fabric handle; the handle travels to the other ranks over the engine's own
// NCCL communicator (ncclBroadcast); every rank imports it, adds its device,
// and — after a barrier, so all devices are members before any memory is
// bound — binds a local physical allocation (the delta + barrier flag) and
// maps both views: unicast (its own memory, read by k_rows) and multicast
// (the address k_deposit_fixed<true> and k_mc_barrier red into).
void mc_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) {
        const char* name = nullptr;
        if (driver().GetErrorName) driver().GetErrorName(r, &name);
        throw Fail{ACO_E_UNSUPPORTED, std::string("NVLS multicast exchange: ") + what + " -> " +
                                          (name ? name : "CUDA driver error")};
    }
}

void nccl_barrier(aco_gpu_ctx* c) {
    int32_t* d = nullptr;
    CK(cudaMalloc(&d, sizeof(int32_t)));
    CK(cudaMemsetAsync(d, 0, sizeof(int32_t), c->stream));
    NK(nccl().AllReduce(d, d, 1, ncclInt32, ncclSum, c->comm, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d);
}

void teardown_multicast(aco_gpu_ctx* c);

// every rank's verdict on a setup step (MIN over the ranks), so that all ranks
// take the same branch and none is left waiting in a collective
bool all_ranks_ok(aco_gpu_ctx* c, bool ok) {
    int32_t* d = nullptr;
    int32_t h = ok ? 1 : 0;
    CK(cudaMalloc(&d, sizeof(int32_t)));
    CK(cudaMemcpyAsync(d, &h, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    NK(nccl().AllReduce(d, d, 1, ncclInt32, ncclMin, c->comm, c->stream));
    CK(cudaMemcpyAsync(&h, d, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d);
    return h == 1;
}

// Returns false (every rank alike, nothing left allocated) when the node
// cannot host the multicast object — no NVSwitch multicast, no fabric-handle
// export (IMEX) — and the caller falls back to the FIXED64 all-reduce, which
// gives the same integers.
bool setup_multicast(aco_gpu_ctx* c) {
    DriverApi& d = driver();
    const bool have = d.MulticastCreate && d.MulticastBindMem && d.MemImportFromShareableHandle &&
                      d.MulticastAddDevice && d.MemCreate && d.MemMap && d.MulticastGetGranularity;
    if (!all_ranks_ok(c, have)) return false;
    const CUmemAllocationHandleType ht = CU_MEM_HANDLE_TYPE_FABRIC;
    const size_t cells = static_cast<size_t>(c->n) * c->P64;
    const size_t want = cells * sizeof(unsigned long long) + 256; // delta + barrier flag
    CUmulticastObjectProp mp{};
    mp.numDevices = static_cast<unsigned int>(c->world);
    mp.handleTypes = ht;
    mp.size = want;
    size_t gran = 0;
    bool ok = d.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS &&
              gran > 0;
    if (!all_ranks_ok(c, ok)) return false;
    c->mc_size = (want + gran - 1) / gran * gran;
    mp.size = c->mc_size;
    // rank 0 creates and exports; the handle (and whether that worked) goes
    // to every rank over the engine's communicator
    struct {
        CUmemFabricHandle fh;
        int32_t ok;
    } msg{};
    if (c->rank == 0) {
        ok = d.MulticastCreate(&c->mc_handle, &mp) == CUDA_SUCCESS;
        if (ok) ok = d.MemExportToShareableHandle(&msg.fh, c->mc_handle, ht, 0) == CUDA_SUCCESS;
        msg.ok = ok ? 1 : 0;
    }
    uint8_t* dh = nullptr;
    CK(cudaMalloc(&dh, sizeof(msg)));
    CK(cudaMemcpyAsync(dh, &msg, sizeof(msg), cudaMemcpyHostToDevice, c->stream));
    NK(nccl().Broadcast(dh, dh, sizeof(msg), ncclUint8, 0, c->comm, c->stream));
    CK(cudaMemcpyAsync(&msg, dh, sizeof(msg), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(dh);
    ok = msg.ok == 1;
    if (ok && c->rank != 0)
        ok = d.MemImportFromShareableHandle(&c->mc_handle, &msg.fh, ht) == CUDA_SUCCESS;
    if (ok) ok = d.MulticastAddDevice(c->mc_handle, static_cast<CUdevice>(c->device)) == CUDA_SUCCESS;
    if (!all_ranks_ok(c, ok)) { // every device joined before any memory is bound
        teardown_multicast(c);
        return false;
    }
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = c->device;
    ap.requestedHandleTypes = ht;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = c->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    ok = d.MemCreate(&c->mc_phys, c->mc_size, &ap, 0) == CUDA_SUCCESS;
    if (ok) ok = d.MulticastBindMem(c->mc_handle, 0, c->mc_phys, 0, c->mc_size, 0) == CUDA_SUCCESS;
    if (ok) ok = d.MemAddressReserve(&c->mc_uc, c->mc_size, gran, 0, 0) == CUDA_SUCCESS;
    if (ok) ok = d.MemMap(c->mc_uc, c->mc_size, 0, c->mc_phys, 0) == CUDA_SUCCESS;
    if (ok) ok = d.MemSetAccess(c->mc_uc, c->mc_size, &acc, 1) == CUDA_SUCCESS;
    if (ok) ok = d.MemAddressReserve(&c->mc_va, c->mc_size, gran, 0, 0) == CUDA_SUCCESS;
    if (ok) ok = d.MemMap(c->mc_va, c->mc_size, 0, c->mc_handle, 0) == CUDA_SUCCESS;
    if (ok) ok = d.MemSetAccess(c->mc_va, c->mc_size, &acc, 1) == CUDA_SUCCESS;
    if (!all_ranks_ok(c, ok)) {
        teardown_multicast(c);
        return false;
    }
    CK(cudaMemsetAsync(reinterpret_cast<void*>(c->mc_uc), 0, c->mc_size, c->stream));
    nccl_barrier(c); // zeroed everywhere before the first red arrives
    c->d_delta_fix = reinterpret_cast<unsigned long long*>(c->mc_uc);
    c->multimem = true;
    return true;
}

void teardown_multicast(aco_gpu_ctx* c) {
    DriverApi& d = driver();
    if (c->mc_va && d.MemUnmap) {
        d.MemUnmap(c->mc_va, c->mc_size);
        d.MemAddressFree(c->mc_va, c->mc_size);
    }
    if (c->mc_uc && d.MemUnmap) {
        d.MemUnmap(c->mc_uc, c->mc_size);
        d.MemAddressFree(c->mc_uc, c->mc_size);
    }
    if (c->mc_handle && c->mc_phys && d.MulticastUnbind)
        d.MulticastUnbind(c->mc_handle, static_cast<CUdevice>(c->device), 0, c->mc_size);
    if (c->mc_phys && d.MemRelease) d.MemRelease(c->mc_phys);
    if (c->mc_handle && d.MemRelease) d.MemRelease(c->mc_handle);
    c->mc_va = c->mc_uc = 0;
    c->mc_phys = c->mc_handle = 0;
    c->d_delta_fix = nullptr;
}

// pow(tau, alpha) for alpha not in {0, 1}: upload the host libm's pow tables
// and prove on this device that libm_pow replays the host's std::pow on a
// spread of pheromone-like arguments (tau0-scaled, down through the
// subnormals, plus random mantissas) — otherwise refuse (ACO_E_UNSUPPORTED),
// never run a silently different pow.
LibmPowTables* upload_pow_tables(cudaStream_t st) {
    LibmPowTables T;
    std::string why;
    if (!read_libm_pow_tables(T, why))
        throw Fail{ACO_E_UNSUPPORTED, "pow(tau, alpha) for alpha not in {0,1}: " + why};
    LibmPowTables* d = nullptr;
    CK(cudaMalloc(&d, sizeof(T)));
    CK(cudaMemcpyAsync(d, &T, sizeof(T), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return d;
}

void pow_self_test(const LibmPowTables* d_tab, double alpha, double tau0, cudaStream_t st) {
    std::vector<double> xs, ys;
    uint64_t s = 0x9E3779B97F4A7C15ull;
    auto next = [&] {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return s;
    };
    for (int e = -1100; e <= 40; ++e) { // tau0 * 2^e and random neighbours
        xs.push_back(std::ldexp(tau0, e));
        const double m = 1.0 + static_cast<double>(next() >> 11) * 0x1.0p-53;
        xs.push_back(std::ldexp(m, e));
    }
    for (int k = 0; k < 2048; ++k) {
        const uint64_t bits = (next() & 0x000FFFFFFFFFFFFFull) | (static_cast<uint64_t>(next() % 0x7FE) << 52);
        double x;
        std::memcpy(&x, &bits, 8);
        xs.push_back(x);
    }
    xs.push_back(0.0);
    xs.push_back(1.0);
    ys.assign(xs.size(), alpha);
    const int cnt = static_cast<int>(xs.size());
    double *dx = nullptr, *dy = nullptr, *dout = nullptr;
    CK(cudaMalloc(&dx, cnt * sizeof(double)));
    CK(cudaMalloc(&dy, cnt * sizeof(double)));
    CK(cudaMalloc(&dout, cnt * sizeof(double)));
    std::vector<double> out(cnt);
    CK(cudaMemcpyAsync(dx, xs.data(), cnt * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dy, ys.data(), cnt * sizeof(double), cudaMemcpyHostToDevice, st));
    k_libm_pow<<<(cnt + 255) / 256, 256, 0, st>>>(dx, dy, cnt, d_tab, dout);
    const cudaError_t le = cudaGetLastError();
    CK(cudaMemcpyAsync(out.data(), dout, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dout);
    if (le != cudaSuccess) throw Fail{ACO_E_CUDA, std::string("k_libm_pow: ") + cudaGetErrorString(le)};
    for (int i = 0; i < cnt; ++i) {
        const double h = host_pow(xs[i], ys[i]);
        if (std::memcmp(&h, &out[i], 8) != 0) {
            char buf[160];
            std::snprintf(buf, sizeof(buf), "device pow(%a, %a) = %a but host libm gives %a", xs[i],
                          ys[i], out[i], h);
            throw Fail{ACO_E_UNSUPPORTED,
                       std::string("pow(tau, alpha) for alpha not in {0,1} cannot be reproduced "
                                   "on this host: ") + buf};
        }
    }
}

// Debug mode: validate this construction's tours on the device and fail
// the call (before any deposit) the way TourBuffer::make would throw.
void check_tours(aco_gpu_ctx* c, const int32_t* d_tours = nullptr, const int64_t* d_len = nullptr,
                 int count = -1, int ant0 = -1) {
    if (!d_tours) {
        d_tours = c->d_tours;
        d_len = c->d_len;
        count = c->mloc;
        ant0 = c->ant_begin;
    }
    if (count <= 0) return;
    const unsigned long long none = ~0ull;
    CK(cudaMemcpyAsync(c->d_verr, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
    const int words = (c->n + 31) / 32;
    const size_t smem = 4 * static_cast<size_t>(words) * sizeof(uint32_t);
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(k_validate_tours, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
    const int grid = std::max(1, std::min((count + 3) / 4, c->num_sms * 8));
    k_validate_tours<<<grid, 128, smem, c->stream>>>(d_tours, c->d_dist, d_len, c->n, c->P64,
                                                      count, c->d_verr);
    check_launch(c, "k_validate_tours");
    unsigned long long e = 0;
    CK(cudaMemcpyAsync(&e, c->d_verr, sizeof(e), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (e == none) return;
    const long long ant = ant0 + static_cast<long long>(e >> 2);
    switch (e & 3) {
    case 1: throw ModelError(Errc::not_closed, "tour does not return to its start (ant " +
                                                   std::to_string(ant) + ")");
    case 2: throw ModelError(Errc::not_a_permutation, "tour is not a permutation of 0.." +
                                                          std::to_string(c->n - 1) + " (ant " +
                                                          std::to_string(ant) + ")");
    default: throw ModelError(Errc::inconsistent_length,
                              "stored length of ant " + std::to_string(ant) + " != recomputed");
    }
}

// construction + tour lengths + iteration stats (no host sync)
void do_construct(aco_gpu_ctx* c) {
    CK(cudaMemsetAsync(c->d_fb, 0, 3 * sizeof(unsigned long long), c->stream));
    CK(cudaEventRecord(c->ev[0], c->stream));
    launch_construct(c);
    CK(cudaEventRecord(c->ev[1], c->stream));
    if (!c->fused_tail) {
        const int warps = 8;
        const int grid = std::max(1, std::min((c->mloc + warps - 1) / warps, c->num_sms * 16));
        int32_t* succ = nullptr;
        int32_t* pred = nullptr;
        if (gather_mode(c)) {
            succ = c->d_succ + static_cast<size_t>(c->rank) * c->n * c->S;
            pred = c->d_pred + static_cast<size_t>(c->rank) * c->n * c->S;
        }
        k_tour_length<<<grid, 32 * warps, 0, c->stream>>>(
            c->d_tours, c->d_dist, c->n, c->P64, c->mloc, c->d_len,
            c->d_inv + static_cast<size_t>(c->rank) * c->S, succ, pred, c->S);
        check_launch(c, "k_tour_length");
    }
    if (c->validate_tours) check_tours(c);
    // unsharded: the stats kernel also maintains best-so-far on device.
    k_iter_stats<<<1, 1024, 0, c->stream>>>(
        c->d_len, c->mloc, c->d_tours, c->n, c->d_stats, c->d_stats + 3, c->d_best,
        c->sharded ? 0 : 1);
    check_launch(c, "k_iter_stats");
    if (c->sharded && !gather_mode(c) && !c->fixed) { // local delta for the all-reduce
        k_deposit_atomic<<<c->num_sms * 8, 256, 0, c->stream>>>(
            c->d_tours, c->d_inv + static_cast<size_t>(c->rank) * c->S, c->n, c->P64, c->mloc,
            c->d_delta);
        check_launch(c, "k_deposit_atomic");
    }
    CK(cudaEventRecord(c->ev[2], c->stream));
}

// exchange + evaporate + deposit + choice (no host sync)
// Fixed-point accumulate: exact int64 delta sums (k_deposit_fixed), then one
// fused evaporate + delta + choice pass (k_rows<DELTA_FIX>).  Sharded: an
// ncclUint64 all-reduce of the delta (wire FIXED64, exact), or — wire
// MULTIMEM, f2 — the deposit's reds go straight to the NVLS multicast object
// (every GPU's delta at once) and a flag barrier through the same object
// replaces the collective.
// nn selection: compact slots + records (k_deposit_nn_fixed), exchanged as
// 2.4 MB + the records instead of the n^2 delta, applied to the local dense
// int64 delta by every rank in the same integers.
void nn_fixed_exchange(aco_gpu_ctx* c, bool shard, const double* inv) {
    const int grid = c->num_sms * 8;
    CK(cudaMemsetAsync(c->d_rec_counts + c->rank, 0, sizeof(unsigned long long), c->stream));
    k_deposit_nn_fixed<<<grid, 256, 0, c->stream>>>(c->d_tours, c->d_qpos, inv, c->n, c->mloc,
                                                     c->cfg.nn, c->d_stats, c->d_dnn_fix, c->d_rec,
                                                     c->d_rec_counts + c->rank);
    check_launch(c, "k_deposit_nn_fixed");
    const size_t slots = static_cast<size_t>(c->n) * c->cfg.nn;
    const DepositRecord* rec = c->d_rec;
    size_t stride = 0;
    int shards = 1;
    if (shard) {
        auto& api = nccl();
        // every rank's record count (one host round trip sizes the all-gather)
        NK(api.AllGather(c->d_rec_counts + c->rank, c->d_rec_counts, 1, ncclUint64, c->comm, c->stream));
        CK(cudaMemcpyAsync(c->h_rec_counts, c->d_rec_counts, c->world * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        unsigned long long mx = 1;
        for (int g = 0; g < c->world; ++g) mx = std::max(mx, c->h_rec_counts[g]);
        if (mx > c->rec_stride) { // grow the gather buffer (rare: fallback-heavy colonies)
            if (c->d_rec_all) CK(cudaFree(c->d_rec_all));
            c->rec_stride = mx + mx / 4;
            CK(cudaMalloc(&c->d_rec_all, c->rec_stride * c->world * sizeof(DepositRecord)));
        }
        NK(api.GroupStart());
        NK(api.AllReduce(c->d_dnn_fix, c->d_dnn_fix, slots, ncclUint64, ncclSum, c->comm, c->stream));
        NK(api.AllGather(c->d_rec, c->d_rec_all, mx * (sizeof(DepositRecord) / 8), ncclUint64, c->comm,
                         c->stream));
        NK(api.GroupEnd());
        rec = c->d_rec_all;
        stride = mx;
        shards = c->world;
    }
    CK(cudaEventRecord(c->ev[3], c->stream));
    k_apply_nn_fixed<<<static_cast<int>(std::min<size_t>((slots + 255) / 256, c->num_sms * 16)), 256, 0,
                       c->stream>>>(c->d_dnn_fix, c->d_nn, c->n, c->cfg.nn, c->P64, c->d_delta_fix);
    check_launch(c, "k_apply_nn_fixed");
    k_apply_records<<<grid, 256, 0, c->stream>>>(rec, shard ? c->d_rec_counts : c->d_rec_counts + c->rank,
                                                  shards, stride, c->P64, c->d_delta_fix);
    check_launch(c, "k_apply_records");
}

void do_update_fixed(aco_gpu_ctx* c) {
    const bool shard = c->sharded && !c->external;
    const int shift = c->key_two_stage ? 0 : c->key_shift;
    k_fixed_scale<<<1, 32, 0, c->stream>>>(c->d_stats, c->m, shift, shard ? 1 : 0);
    check_launch(c, "k_fixed_scale");
    const double* inv = c->d_inv + static_cast<size_t>(c->rank) * c->S;
    if (c->d_dnn_fix) {
        nn_fixed_exchange(c, shard, inv);
    } else if (c->multimem) {
        k_deposit_fixed<true><<<c->num_sms * 8, 256, 0, c->stream>>>(
            c->d_tours, inv, c->n, c->P64, c->mloc, c->d_stats,
            reinterpret_cast<unsigned long long*>(c->mc_va));
        check_launch(c, "k_deposit_fixed<multimem>");
        const size_t flag_off = static_cast<size_t>(c->n) * c->P64 * sizeof(unsigned long long);
        ++c->mc_epoch;
        k_mc_barrier<<<1, 32, 0, c->stream>>>(
            reinterpret_cast<unsigned long long*>(c->mc_va + flag_off),
            reinterpret_cast<const unsigned long long*>(c->mc_uc + flag_off),
            c->mc_epoch * static_cast<unsigned long long>(c->world));
        check_launch(c, "k_mc_barrier");
    } else {
        k_deposit_fixed<false><<<c->num_sms * 8, 256, 0, c->stream>>>(
            c->d_tours, inv, c->n, c->P64, c->mloc, c->d_stats, c->d_delta_fix);
        check_launch(c, "k_deposit_fixed");
        if (shard) {
            const size_t cells = static_cast<size_t>(c->n) * c->P64;
            NK(nccl().AllReduce(c->d_delta_fix, c->d_delta_fix, cells, ncclUint64, ncclSum, c->comm,
                                c->stream));
        }
    }
    if (!c->d_dnn_fix) CK(cudaEventRecord(c->ev[3], c->stream));
    launch_rows(c, MODE_DELTA_FIX);
    CK(cudaEventRecord(c->ev[4], c->stream));
    CK(cudaEventRecord(c->ev[5], c->stream));
}

void do_update(aco_gpu_ctx* c) {
    const double keep = 1.0 - c->cfg.rho;
    if (c->fixed) {
        do_update_fixed(c);
        return;
    }
    if (c->sharded && !c->external) {
        auto& api = nccl();
        if (gather_mode(c) && c->row_shard) {
            // rank q needs, from every rank g, g's succ/pred rows of q's row
            // block: [g][q*B .. q*B+rows_q) of the [world][n][S] tables
            const size_t blk = static_cast<size_t>(c->n) * c->S;
            const int B = c->row_blk;
            auto rows_of = [&](int q) { return std::max(0, std::min(c->n, (q + 1) * B) - q * B); };
            NK(api.GroupStart());
            for (int q = 0; q < c->world; ++q) {
                if (q == c->rank) continue;
                const size_t out_off = c->rank * blk + static_cast<size_t>(q) * B * c->S;
                const size_t out_cnt = static_cast<size_t>(rows_of(q)) * c->S;
                const size_t in_off = q * blk + static_cast<size_t>(c->rank) * B * c->S;
                const size_t in_cnt = static_cast<size_t>(rows_of(c->rank)) * c->S;
                if (out_cnt) {
                    NK(api.Send(c->d_succ + out_off, out_cnt, ncclInt32, q, c->comm, c->stream));
                    NK(api.Send(c->d_pred + out_off, out_cnt, ncclInt32, q, c->comm, c->stream));
                }
                if (in_cnt) {
                    NK(api.Recv(c->d_succ + in_off, in_cnt, ncclInt32, q, c->comm, c->stream));
                    NK(api.Recv(c->d_pred + in_off, in_cnt, ncclInt32, q, c->comm, c->stream));
                }
            }
            NK(api.GroupEnd());
            // (the 1/C_k all-gather in its own call, not grouped with p2p)
            NK(api.AllGather(c->d_inv + static_cast<size_t>(c->rank) * c->S, c->d_inv, c->S,
                             ncclFloat64, c->comm, c->stream));
            CK(cudaEventRecord(c->ev[3], c->stream));
            launch_rows(c, MODE_FOLD_OWN);
            const size_t dblk = static_cast<size_t>(B) * c->P64;
            NK(api.AllGather(c->d_delta + c->rank * dblk, c->d_delta, dblk, ncclFloat64, c->comm,
                             c->stream));
            launch_rows(c, MODE_APPLY);
            CK(cudaEventRecord(c->ev[4], c->stream));
            CK(cudaEventRecord(c->ev[5], c->stream));
            return;
        } else if (gather_mode(c)) {
            const size_t blk = static_cast<size_t>(c->n) * c->S;
            NK(api.GroupStart());
            NK(api.AllGather(c->d_succ + c->rank * blk, c->d_succ, blk, ncclInt32, c->comm, c->stream));
            NK(api.AllGather(c->d_pred + c->rank * blk, c->d_pred, blk, ncclInt32, c->comm, c->stream));
            NK(api.AllGather(c->d_inv + static_cast<size_t>(c->rank) * c->S, c->d_inv, c->S,
                             ncclFloat64, c->comm, c->stream));
            NK(api.GroupEnd());
        } else {
            const size_t cells = static_cast<size_t>(c->n) * c->P64;
            if (c->d_delta32) {
                k_delta_pack<<<c->num_sms * 8, 256, 0, c->stream>>>(c->d_delta, c->d_delta32, cells / 2);
                check_launch(c, "k_delta_pack");
                NK(api.AllReduce(c->d_delta32, c->d_delta32, cells, ncclFloat32, ncclSum, c->comm,
                                 c->stream));
            } else {
                NK(api.AllReduce(c->d_delta, c->d_delta, cells, ncclFloat64, ncclSum, c->comm,
                                 c->stream));
            }
        }
    }
    CK(cudaEventRecord(c->ev[3], c->stream));
    if (gather_mode(c) && c->external && c->folded) { // aco_gpu_fold ran: apply the gathered delta rows
        c->folded = false;
        launch_rows(c, MODE_APPLY);
        CK(cudaEventRecord(c->ev[4], c->stream));
    } else if (gather_mode(c)) {
        launch_rows(c, MODE_GATHER);
        CK(cudaEventRecord(c->ev[4], c->stream));
    } else if (c->sharded) {
        launch_rows(c, (c->d_delta32 && !c->external) ? MODE_DELTA32 : MODE_DELTA);
        CK(cudaEventRecord(c->ev[4], c->stream));
    } else {
        const size_t count2 = static_cast<size_t>(c->n) * c->P64 / 2;
        if (c->sym) {
            // evaporation fused into k_rows<MODE_DELTA_SYM>; one red per edge
            CK(cudaMemsetAsync(c->d_delta, 0, static_cast<size_t>(c->n) * c->P64 * sizeof(double), c->stream));
            k_deposit_sym<<<c->num_sms * 8, 256, 0, c->stream>>>(c->d_tours, c->d_inv, c->n, c->P64,
                                                                 c->mloc, c->d_delta);
            check_launch(c, "k_deposit_sym");
            CK(cudaEventRecord(c->ev[4], c->stream));
            launch_rows(c, MODE_DELTA_SYM);
            CK(cudaEventRecord(c->ev[5], c->stream));
            return;
        }
        k_evaporate<<<c->num_sms * 8, 256, 0, c->stream>>>(c->d_tau, count2, keep);
        check_launch(c, "k_evaporate");
        if (c->d_dnn) { // nn selection: list edges through the compact slots
            k_deposit_nn<<<c->num_sms * 8, 256, 0, c->stream>>>(c->d_tours, c->d_qpos, c->d_inv, c->n,
                                                                c->P64, c->mloc, c->cfg.nn, c->d_dnn,
                                                                c->d_tau);
            check_launch(c, "k_deposit_nn");
            const size_t slots = static_cast<size_t>(c->n) * c->cfg.nn;
            k_apply_nn<<<static_cast<int>(std::min<size_t>((slots + 255) / 256, c->num_sms * 16)), 256, 0,
                         c->stream>>>(c->d_dnn, c->d_nn, c->n, c->cfg.nn, c->P64, c->d_tau);
            check_launch(c, "k_apply_nn");
        } else {
            k_deposit_atomic<<<c->num_sms * 8, 256, 0, c->stream>>>(c->d_tours, c->d_inv, c->n, c->P64,
                                                                    c->mloc, c->d_tau);
            check_launch(c, "k_deposit_atomic");
        }
        CK(cudaEventRecord(c->ev[4], c->stream));
        launch_rows(c, MODE_CHOICE);
    }
    CK(cudaEventRecord(c->ev[5], c->stream));
}

float ev_ms(aco_gpu_ctx* c, int a, int b) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]));
    return ms;
}

// Sharded (NCCL) statistics, enqueued on the engine stream with no host
// synchronisation: key MIN + sum SUM all-reduces, the owner's tour
// replicated by an all-reduce MAX, best-so-far updated on the device.
void enqueue_shard_stats(aco_gpu_ctx* c) {
    auto& api = nccl();
    long long* s = c->d_stats;
    const int shift = c->key_two_stage ? 0 : c->key_shift;
    k_shard_key<<<1, 32, 0, c->stream>>>(s, c->ant_begin, c->mloc, shift);
    check_launch(c, "k_shard_key");
    NK(api.GroupStart());
    NK(api.AllReduce(s + 4, s + 4, 1, ncclInt64, ncclMin, c->comm, c->stream));
    NK(api.AllReduce(s + 6, s + 6, 1, ncclInt64, ncclSum, c->comm, c->stream));
    NK(api.GroupEnd());
    if (c->key_two_stage) { // s[5] = lowest global ant among the ranks holding min length
        k_shard_ant<<<1, 32, 0, c->stream>>>(s, c->ant_begin, c->mloc);
        check_launch(c, "k_shard_ant");
        NK(api.AllReduce(s + 5, s + 5, 1, ncclInt64, ncclMin, c->comm, c->stream));
    }
    k_owner_tour<<<std::max(1, (c->n + 256) / 256), 256, 0, c->stream>>>(
        s, c->d_tours, c->n, c->ant_begin, c->ant_end, c->d_tourbuf, shift);
    check_launch(c, "k_owner_tour");
    NK(api.AllReduce(c->d_tourbuf, c->d_tourbuf, c->n + 1, ncclInt32, ncclMax, c->comm, c->stream));
    k_best_update<<<1, 1024, 0, c->stream>>>(s, c->d_tourbuf, c->n, c->d_best, shift);
    check_launch(c, "k_best_update");
}

// Fills the record from h_stats[0..7] (copied from d_stats after the stream
// synchronised).  Sharded: the reduced key / sum and the device best-so-far;
// otherwise (and in external mode) this shard's own statistics.
void finish_stats(aco_gpu_ctx* c, aco_gpu_iter_record* rec) {
    if (c->sharded && !c->external) {
        rec->best_length = c->key_two_stage ? c->h_stats[4] : c->h_stats[4] >> c->key_shift;
        rec->mean_length = static_cast<double>(c->h_stats[6]) / static_cast<double>(c->m);
        c->best_so_far = c->h_stats[3];
    } else {
        rec->best_length = c->h_stats[0];
        rec->mean_length = static_cast<double>(c->h_stats[2]) / static_cast<double>(c->mloc);
        c->best_so_far = std::min<int64_t>(c->best_so_far, c->h_stats[0]);
    }
}

void fill_common(aco_gpu_ctx* c, aco_gpu_iter_record* rec) {
    rec->iteration = c->iteration + 1;
    predicted_access_cost(c->cfg.deposit, c->n, c->m, c->cfg.theta, rec->ledger);
}

} // namespace

// ===========================================================================
extern "C" {

const char* aco_errc_name(int s) {
    static const char* names[] = {"ok", "missing_field", "unsupported_edge_weight_type",
                                  "malformed_coord", "dimension_mismatch", "index_out_of_range",
                                  "overflow", "invalid_length", "not_a_permutation", "not_closed",
                                  "all_visited", "inconsistent_length", "io_error", "config_error"};
    if (s >= 0 && s <= 13) return names[s];
    if (s == ACO_E_CUDA) return "cuda_error";
    if (s == ACO_E_NCCL) return "nccl_error";
    if (s == ACO_E_UNSUPPORTED) return "unsupported";
    return "unknown";
}

const char* aco_last_error(void) { return g_host_err.c_str(); }

aco_status aco_parse_instance(const char* text, int32_t* dimension, int32_t* ewt, double* xs,
                              double* ys, int32_t capacity, char* name, int32_t name_capacity) {
    return guard_ctx(nullptr, [&] {
        Instance in;
        parse_instance(text ? std::string_view(text) : std::string_view(), in);
        *dimension = in.dimension;
        if (ewt) *ewt = in.edge_weight_type;
        if (xs && ys && capacity >= in.dimension) {
            std::copy(in.xs.begin(), in.xs.end(), xs);
            std::copy(in.ys.begin(), in.ys.end(), ys);
        }
        if (name && name_capacity > 0) {
            std::snprintf(name, static_cast<size_t>(name_capacity), "%s", in.name.c_str());
        }
    });
}

aco_status aco_parse_tour(const char* text, int32_t* tour, int32_t capacity, int32_t* length) {
    return guard_ctx(nullptr, [&] {
        const auto t = parse_tour(text ? std::string_view(text) : std::string_view());
        *length = static_cast<int32_t>(t.size());
        for (int i = 0; i < static_cast<int>(t.size()) && i < capacity; ++i) tour[i] = t[i];
    });
}

aco_status aco_build_distances(int32_t n, const double* xs, const double* ys, int32_t ewt,
                               int32_t* dist) {
    return guard_ctx(nullptr, [&] { build_distances(n, xs, ys, ewt, dist); });
}

aco_status aco_build_nn_lists(int32_t n, const int32_t* dist, int32_t nn, int32_t* out) {
    return guard_ctx(nullptr, [&] { build_nn_lists(n, dist, nn, out); });
}

aco_status aco_greedy_tour_length(int32_t n, const int32_t* dist, int64_t* out) {
    return guard_ctx(nullptr, [&] { *out = greedy_tour_length(n, dist); });
}

aco_status aco_tour_length(int32_t n, const int32_t* dist, const int32_t* tour, int32_t len,
                           int64_t* out) {
    return guard_ctx(nullptr, [&] { *out = tour_length(n, dist, tour, len); });
}

aco_status aco_predicted_access_cost(int32_t deposit, int32_t n, int32_t m, int32_t theta,
                                     double out[4]) {
    return guard_ctx(nullptr, [&] {
        if (deposit < 0 || deposit > 3) throw ModelError(Errc::config_error, "unknown deposit strategy");
        predicted_access_cost(deposit, n, m, theta, out);
    });
}

aco_status aco_validate_parameters(double alpha, double beta, double rho, int32_t m, int32_t nn,
                                   int32_t iterations, int32_t tile_size, int32_t n,
                                   int32_t nn_selected) {
    return guard_ctx(nullptr, [&] {
        Config c;
        c.n = n;
        c.m = m;
        c.nn = nn;
        c.theta = tile_size;
        c.iterations = iterations;
        c.selection = nn_selected ? ACO_SEL_NN : ACO_SEL_ROULETTE;
        c.alpha = alpha;
        c.beta = beta;
        c.rho = rho;
        validate(c);
    });
}

double aco_uniform_at(uint64_t seed, uint32_t iteration, uint32_t ant, uint32_t step,
                      uint32_t draw) {
    return philox_uniform(seed, iteration, ant, step, draw);
}

aco_status aco_gpu_nccl_unique_id(uint8_t out[128]) {
    return guard_ctx(nullptr, [&] {
        auto& api = nccl();
        if (!api.GetUniqueId) throw Fail{ACO_E_NCCL, "libnccl.so.2 not found"};
        ncclUniqueId id;
        NK(api.GetUniqueId(&id));
        static_assert(sizeof(id) == 128, "nccl id size");
        std::memcpy(out, &id, 128);
    });
}

aco_status aco_gpu_create(const aco_gpu_params* prm, const int32_t* dist, aco_gpu_ctx** out) {
    if (!out) return ACO_E_CONFIG_ERROR;
    *out = nullptr;
    auto* c = new aco_gpu_ctx;
    const aco_status st = guard_ctx(c, [&] {
        if (!prm || !dist) throw ModelError(Errc::config_error, "params and dist are required");
        if (prm->n < 2) throw ModelError(Errc::dimension_mismatch, "n must be at least 2");
        c->cfg.n = c->n = prm->n;
        c->cfg.m = prm->m == 0 ? prm->n : prm->m; // engine.hpp:60
        c->cfg.nn = prm->nn;
        c->cfg.theta = prm->theta;
        c->cfg.selection = prm->selection;
        c->cfg.deposit = prm->deposit;
        c->cfg.alpha = prm->alpha;
        c->cfg.beta = prm->beta;
        c->cfg.rho = prm->rho;
        validate(c->cfg);
        if (c->cfg.selection == ACO_SEL_NN && c->cfg.nn > 64)
            throw Fail{ACO_E_UNSUPPORTED, "nn lists longer than 64 are not supported"};
        if (c->cfg.m < 1) throw ModelError(Errc::config_error, "ant count must be >= 1");
        c->m = c->cfg.m;
        c->seed = prm->seed;
        c->random_start = prm->random_start;
        c->stream_kind = prm->stream == ACO_STREAM_FP64 ? ACO_STREAM_FP64 : ACO_STREAM_FP32;
        c->world = prm->world > 1 ? prm->world : 1;
        c->rank = c->world > 1 ? prm->rank : 0;
        if (c->rank < 0 || c->rank >= c->world) throw ModelError(Errc::config_error, "bad rank");
        c->S = (c->m + c->world - 1) / c->world;
        if (c->world == 1 && (prm->ant_begin != 0 || prm->ant_end != 0)) {
            if (!(0 <= prm->ant_begin && prm->ant_begin < prm->ant_end && prm->ant_end <= c->m))
                throw ModelError(Errc::config_error, "bad ant range");
            c->ant_begin = prm->ant_begin;
            c->ant_end = prm->ant_end;
            c->S = c->ant_end - c->ant_begin;
        } else {
            c->ant_begin = std::min(c->m, c->rank * c->S);
            c->ant_end = std::min(c->m, (c->rank + 1) * c->S);
        }
        c->mloc = c->ant_end - c->ant_begin;
        c->device = prm->device;
        c->validate_tours = prm->validate_tours != 0;
        {
            // world > 1 with a zero id: external exchange (the caller runs
            // the collectives); world == 1 with an id: the sharded protocol on
            // a one-rank NCCL communicator (exercises the exchange path)
            bool zero = true;
            for (int i = 0; i < 128; ++i) zero = zero && prm->nccl_id[i] == 0;
            c->sharded = c->world > 1 || !zero;
            c->external = c->world > 1 && zero;
            if (c->world == 1 && !zero && (prm->ant_begin != 0 || prm->ant_end != 0))
                throw ModelError(Errc::config_error, "an ant range and an NCCL id exclude each other");
        }

        // host model: distances, eta^beta table, tau0, nn lists
        const int n = c->n;
        for (size_t i = 0; i < static_cast<size_t>(n) * n; ++i) {
            if (dist[i] < 0) throw ModelError(Errc::overflow, "negative distance");
            c->max_d = std::max<int64_t>(c->max_d, dist[i]);
        }
        if (c->max_d > 0 && static_cast<int64_t>(n) > std::numeric_limits<int64_t>::max() / c->max_d)
            throw ModelError(Errc::overflow, "tour lengths would overflow 64-bit range");
        c->tau0 = static_cast<double>(c->m) / static_cast<double>(greedy_tour_length(n, dist));
        std::vector<int32_t> nn_host;
        if (c->cfg.selection == ACO_SEL_NN) {
            nn_host.resize(static_cast<size_t>(n) * c->cfg.nn);
            build_nn_lists(n, dist, c->cfg.nn, nn_host.data());
        }

        // device
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (c->device < 0 || c->device >= ndev) throw Fail{ACO_E_CUDA, "no such CUDA device"};
        CK(cudaSetDevice(c->device));
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
        choose_stream_layout(c);
        c->P64 = round_up(n, 32);
        const size_t cells = static_cast<size_t>(n) * c->P64;
        CK(cudaMalloc(&c->d_dist, cells * sizeof(int32_t)));
        CK(cudaMemset(c->d_dist, 0, cells * sizeof(int32_t)));
        CK(cudaMemcpy2D(c->d_dist, c->P64 * sizeof(int32_t), dist, n * sizeof(int32_t),
                        n * sizeof(int32_t), n, cudaMemcpyHostToDevice));
        if (c->max_d <= (1 << 25)) {
            const std::vector<double> lut = eta_beta_table(c->max_d, c->cfg.beta);
            CK(cudaMalloc(&c->d_lut, lut.size() * sizeof(double)));
            CK(cudaMemcpy(c->d_lut, lut.data(), lut.size() * sizeof(double), cudaMemcpyHostToDevice));
        } else {
            // very long edges: a dense eta^beta matrix instead of a table
            std::vector<double> et(cells, 0.0);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    const int32_t d = dist[static_cast<size_t>(i) * n + j];
                    const double eta = d > 0 ? 1.0 / d : 1.0;
                    et[static_cast<size_t>(i) * c->P64 + j] = std::pow(eta, c->cfg.beta);
                }
            CK(cudaMalloc(&c->d_etab, cells * sizeof(double)));
            CK(cudaMemcpy(c->d_etab, et.data(), cells * sizeof(double), cudaMemcpyHostToDevice));
        }
        CK(cudaMalloc(&c->d_tau, cells * sizeof(double)));
        CK(cudaMemset(c->d_tau, 0, cells * sizeof(double)));
        CK(cudaMalloc(&c->d_choice, cells * sizeof(double)));
        CK(cudaMemset(c->d_choice, 0, cells * sizeof(double)));
        const size_t wcells = static_cast<size_t>(n) * c->PW;
        if (c->cfg.selection == ACO_SEL_ROULETTE && c->PW > 0) {
            if (c->stream_kind == ACO_STREAM_FP32) {
                CK(cudaMalloc(&c->d_choice32, wcells * sizeof(float)));
                CK(cudaMemset(c->d_choice32, 0, wcells * sizeof(float)));
            } else {
                CK(cudaMalloc(&c->d_choice_p64, wcells * sizeof(double)));
                CK(cudaMemset(c->d_choice_p64, 0, wcells * sizeof(double)));
            }
        }
        CK(cudaMalloc(&c->d_scale, n * sizeof(int32_t)));
        CK(cudaMemset(c->d_scale, 0, n * sizeof(int32_t)));
        if (!nn_host.empty()) {
            CK(cudaMalloc(&c->d_nn, nn_host.size() * sizeof(int32_t)));
            CK(cudaMemcpy(c->d_nn, nn_host.data(), nn_host.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
            CK(cudaMalloc(&c->d_choice_nn, nn_host.size() * sizeof(double)));
            if (c->cfg.nn <= 32) {
                CK(cudaMalloc(&c->d_choice_nn32, nn_host.size() * sizeof(int2)));
                CK(cudaMalloc(&c->d_nn_scale, n * sizeof(int32_t)));
            }
            const char* tke = std::getenv("ACO_NN_TOPK"); // "0" disables the argmax cache
            if (!(tke && tke[0] == '0'))
                CK(cudaMalloc(&c->d_topk, static_cast<size_t>(n) * kTopK * sizeof(int32_t)));
        }
        const size_t ml = std::max(1, c->mloc);
        if (prm->wire < ACO_WIRE_FP64 || prm->wire > ACO_WIRE_MULTIMEM)
            throw ModelError(Errc::config_error, "unknown wire");
        c->fixed = c->cfg.deposit == ACO_DEP_ACCUMULATE &&
                   (prm->wire == ACO_WIRE_FIXED64 || prm->wire == ACO_WIRE_MULTIMEM);
        if (c->fixed && c->external)
            throw ModelError(Errc::config_error,
                             "fixed-point / multimem exchange needs the engine's own NCCL communicator");
        {
            // nn + accumulate on one context: compact list-edge deposit
            // (k_deposit_nn); ACO_NN_COMPACT=0 keeps the plain scatter
            const char* cmp = std::getenv("ACO_NN_COMPACT");
            if (c->cfg.selection == ACO_SEL_NN && c->cfg.deposit == ACO_DEP_ACCUMULATE && !c->sharded &&
                !c->fixed && !(cmp && cmp[0] == '0')) {
                CK(cudaMalloc(&c->d_qpos, ml * n));
                CK(cudaMemset(c->d_qpos, 255, ml * n));
                CK(cudaMalloc(&c->d_dnn, static_cast<size_t>(n) * c->cfg.nn * sizeof(double)));
                CK(cudaMemset(c->d_dnn, 0, static_cast<size_t>(n) * c->cfg.nn * sizeof(double)));
            }
        }
        CK(cudaMalloc(&c->d_tours, ml * (n + 1) * sizeof(int32_t)));
        CK(cudaMemset(c->d_tours, 0, ml * (n + 1) * sizeof(int32_t)));
        CK(cudaMalloc(&c->d_len, ml * sizeof(int64_t)));
        CK(cudaMalloc(&c->d_inv, static_cast<size_t>(c->world) * c->S * sizeof(double)));
        CK(cudaMemset(c->d_inv, 0, static_cast<size_t>(c->world) * c->S * sizeof(double)));
        if (c->cfg.deposit != ACO_DEP_ACCUMULATE) {
            // zeroed: a shard block not yet exchanged folds +0.0 into column 0
            const size_t sp = static_cast<size_t>(c->world) * n * c->S;
            CK(cudaMalloc(&c->d_succ, sp * sizeof(int32_t)));
            CK(cudaMalloc(&c->d_pred, sp * sizeof(int32_t)));
            CK(cudaMemset(c->d_succ, 0, sp * sizeof(int32_t)));
            CK(cudaMemset(c->d_pred, 0, sp * sizeof(int32_t)));
        }
        const char* gsplit = std::getenv("ACO_GATHER_SPLIT");
        const bool warp_gather = c->cfg.deposit != ACO_DEP_ACCUMULATE &&
                                 static_cast<size_t>(c->P64) * sizeof(double) + 64 * sizeof(double) <= 32 * 1024;
        // nn + fixed: compact slots + records exchange; the dense int64 delta
        // stays local (no multicast needed — the exchange is already small)
        const bool nn_fixed = c->fixed && c->cfg.selection == ACO_SEL_NN;
        // (ACO_MC_ONE_RANK=1: also attempt the multicast object on a one-rank
        // communicator — a test hook for the agreement / fallback path, since
        // cuMulticastCreate refuses a one-device object)
        const char* mc1 = std::getenv("ACO_MC_ONE_RANK");
        const bool mc_wanted = c->fixed && prm->wire == ACO_WIRE_MULTIMEM && !nn_fixed && c->sharded &&
                               !c->external && (c->world > 1 || (mc1 && mc1[0] == '1'));
        if (nn_fixed) {
            const size_t ml2 = std::max(1, c->mloc);
            CK(cudaMalloc(&c->d_qpos, ml2 * n));
            CK(cudaMemset(c->d_qpos, 255, ml2 * n));
            const size_t slots = static_cast<size_t>(n) * c->cfg.nn;
            CK(cudaMalloc(&c->d_dnn_fix, slots * sizeof(unsigned long long)));
            CK(cudaMemset(c->d_dnn_fix, 0, slots * sizeof(unsigned long long)));
            CK(cudaMalloc(&c->d_rec, ml2 * n * sizeof(DepositRecord)));
            CK(cudaMalloc(&c->d_rec_counts, c->world * sizeof(unsigned long long)));
            CK(cudaMemset(c->d_rec_counts, 0, c->world * sizeof(unsigned long long)));
            CK(cudaMallocHost(&c->h_rec_counts, c->world * sizeof(unsigned long long)));
        }
        if (c->fixed && !mc_wanted) { // exact int64 delta (one GPU, or the ncclUint64 all-reduce)
            CK(cudaMalloc(&c->d_delta_fix, cells * sizeof(unsigned long long)));
            CK(cudaMemset(c->d_delta_fix, 0, cells * sizeof(unsigned long long)));
        }
        // Gather deposit over several ranks: each folds only its block of
        // ceil(n/world) rows (the succ/pred rows of that block arrive from every
        // rank by send/recv instead of an all-gather of the whole tables) and
        // the delta rows are all-gathered (ACO_ROW_SHARD=0: replicated fold).
        const char* rsh = std::getenv("ACO_ROW_SHARD");
        c->row_shard = c->sharded && c->world > 1 && warp_gather && !(gsplit && gsplit[0] == '0') &&
                       !(rsh && rsh[0] == '0');
        c->row_blk = c->row_shard ? (n + c->world - 1) / c->world : n;
        c->sym = ACO_SYM_DEPOSIT && !c->sharded && !c->fixed && c->cfg.deposit == ACO_DEP_ACCUMULATE &&
                 c->cfg.selection != ACO_SEL_NN;
        if ((c->sharded && c->cfg.deposit == ACO_DEP_ACCUMULATE && !c->fixed) || c->sym ||
            (warp_gather && !(gsplit && gsplit[0] == '0'))) {
            // row-sharded: world row blocks of row_blk rows (the last one padded)
            const size_t dcells = std::max(cells, static_cast<size_t>(c->world) * c->row_blk * c->P64);
            CK(cudaMalloc(&c->d_delta, dcells * sizeof(double)));
            CK(cudaMemset(c->d_delta, 0, dcells * sizeof(double)));
            // fp32 wire only on request (aco_gpu_params::wire): the default
            // all-reduces the fp64 delta, so tours do not depend on G
            if (c->sharded && !c->external && c->cfg.deposit == ACO_DEP_ACCUMULATE &&
                prm->wire == ACO_WIRE_FP32)
                CK(cudaMalloc(&c->d_delta32, cells * sizeof(float)));
        }
        CK(cudaMalloc(&c->d_stats, 8 * sizeof(long long)));
        const long long init_stats[8] = {0, 0, 0, LLONG_MAX, 0, 0, 0, 0};
        CK(cudaMemcpy(c->d_stats, init_stats, sizeof(init_stats), cudaMemcpyHostToDevice));
        CK(cudaMalloc(&c->d_best, (n + 1) * sizeof(int32_t)));
        CK(cudaMemset(c->d_best, 0, (n + 1) * sizeof(int32_t)));
        CK(cudaMalloc(&c->d_verr, sizeof(unsigned long long)));
        CK(cudaMalloc(&c->d_fb, 3 * sizeof(unsigned long long)));
        CK(cudaMemset(c->d_fb, 0, 3 * sizeof(unsigned long long)));
#if ACO_TIMING
        CK(cudaMalloc(&c->d_timing, 8 * sizeof(unsigned long long)));
        CK(cudaMemset(c->d_timing, 0, 8 * sizeof(unsigned long long)));
#endif
        CK(cudaMallocHost(&c->h_stats, 16 * sizeof(long long)));
        if (c->sharded) {
            // iteration-best key: (length << key_shift) | global ant in ONE
            // MIN all-reduce when every tour length fits (length < n * max_d);
            // otherwise two MIN all-reduces, the length and then the lowest
            // ant among the ranks that hold it (engine.hpp:117-129 tie rule)
            c->key_shift = 1;
            while ((int64_t{1} << c->key_shift) < c->m) ++c->key_shift;
            const int64_t max_len = static_cast<int64_t>(n) * std::max<int64_t>(c->max_d, 1);
            c->key_two_stage = c->key_shift >= 62 || max_len >= (int64_t{1} << (62 - c->key_shift));
            CK(cudaMalloc(&c->d_tourbuf, (n + 1) * sizeof(int32_t)));
        }

        if (c->sharded && !c->external) {
            auto& api = nccl();
            if (!api.CommInitRank) throw Fail{ACO_E_NCCL, "libnccl.so.2 not found"};
            if (!api.Send || !api.Recv) c->row_shard = false; // pre-p2p NCCL: replicated fold
            ncclUniqueId id;
            std::memcpy(&id, prm->nccl_id, sizeof(id));
            NK(api.CommInitRank(&c->comm, c->world, id, c->rank));
            if (mc_wanted && !setup_multicast(c)) {
                // no multicast object on this node: the FIXED64 all-reduce of
                // the same exact int64 sums (aco_gpu_describe says which ran)
                CK(cudaMalloc(&c->d_delta_fix, cells * sizeof(unsigned long long)));
                CK(cudaMemset(c->d_delta_fix, 0, cells * sizeof(unsigned long long)));
                c->mc_fallback = true;
            }
        }

        if (c->cfg.alpha != 0.0 && c->cfg.alpha != 1.0) {
            c->d_powtab = upload_pow_tables(c->stream);
            pow_self_test(c->d_powtab, c->cfg.alpha, c->tau0, c->stream);
        }

        // tau0 everywhere (diagonal included, model.hpp:258-262), then choice
        k_fill<<<c->num_sms * 4, 256, 0, c->stream>>>(c->d_tau, cells, c->tau0);
        check_launch(c, "k_fill");
        // pad columns stay zero
        if (c->P64 != n)
            CK(cudaMemset2DAsync(c->d_tau + n, c->P64 * sizeof(double), 0,
                                 (c->P64 - n) * sizeof(double), n, c->stream));
        launch_rows(c, MODE_CHOICE);
        CK(cudaStreamSynchronize(c->stream));
    });
    if (st != ACO_OK) {
        aco_gpu_destroy(c);
        return st;
    }
    *out = c;
    return ACO_OK;
}

void aco_gpu_destroy(aco_gpu_ctx* c) {
    if (!c) return;
#if ACO_TIMING
    if (c->d_timing) {
        unsigned long long h[8];
        cudaMemcpy(h, c->d_timing, sizeof(h), cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "ACO_TIMING cycles per ant-step (all iterations): pass1 %.0f scan %.0f walk %.0f cert %.0f fallback %.0f book %.0f tmawait %.0f\n",
                     h[0] / (double)c->iteration / c->mloc / (c->n - 1), h[1] / (double)c->iteration / c->mloc / (c->n - 1),
                     h[2] / (double)c->iteration / c->mloc / (c->n - 1), h[3] / (double)c->iteration / c->mloc / (c->n - 1),
                     h[4] / (double)c->iteration / c->mloc / (c->n - 1), h[5] / (double)c->iteration / c->mloc / (c->n - 1),
                     h[6] / (double)c->iteration / c->mloc / (c->n - 1));
        cudaFree(c->d_timing);
    }
#endif
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    if (c->multimem) teardown_multicast(c);
    if (c->comm && nccl().CommDestroy) nccl().CommDestroy(c->comm);
    void* bufs[] = {c->d_choice_nn, c->d_choice_nn32, c->d_nn_scale, c->d_topk, c->d_dist, c->d_lut, c->d_etab, c->d_tau, c->d_choice, c->d_choice32,
                    c->d_choice_p64, c->d_scale, c->d_nn, c->d_tours, c->d_len, c->d_inv,
                    c->d_succ, c->d_pred, c->d_delta, c->d_delta32, c->d_stats, c->d_best, c->d_fb, c->d_tourbuf, c->d_verr, c->d_powtab,
                    c->d_qpos, c->d_dnn, c->d_delta_fix, c->d_dnn_fix, c->d_rec, c->d_rec_all,
                    c->d_rec_counts, c->d_relay_flag, c->d_relay_cur, c->d_relay_tabu};
    for (void* b : bufs)
        if (b) cudaFree(b);
    if (c->h_stats) cudaFreeHost(c->h_stats);
    if (c->h_rec_counts) cudaFreeHost(c->h_rec_counts);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
}

const char* aco_gpu_last_error(const aco_gpu_ctx* c) { return c ? c->err.c_str() : g_host_err.c_str(); }

int64_t aco_gpu_launch_count(const aco_gpu_ctx* c) { return c ? c->launches : 0; }

int32_t aco_gpu_describe(const aco_gpu_ctx* c, char* buf, int32_t len) {
    if (!c) return 0;
    std::string d = c->construct_desc;
    if (c->multimem) d += " exchange=multimem";
    else if (c->mc_fallback) d += " exchange=fixed64 (multicast unavailable)";
    if (c->cfg.selection == ACO_SEL_NN)
        d += " argmax_fallbacks=" + std::to_string(c->last_fb[1]) + " full_row_scans=" +
             std::to_string(c->last_fb[0]) + (c->d_topk ? " topk=" + std::to_string(kTopK) : " topk=off");
    if (buf && len > 0) {
        const size_t k = std::min(d.size(), static_cast<size_t>(len - 1));
        std::memcpy(buf, d.data(), k);
        buf[k] = 0;
    }
    return static_cast<int32_t>(d.size());
}

void* aco_gpu_stream(aco_gpu_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

aco_status aco_gpu_exchange_buffers(aco_gpu_ctx* c, void** succ, void** pred, void** inv,
                                    void** delta, int32_t* shard_stride, int32_t* P64) {
    if (!c) return ACO_E_CONFIG_ERROR;
    if (succ) *succ = c->d_succ;
    if (pred) *pred = c->d_pred;
    if (inv) *inv = c->d_inv;
    if (delta) *delta = c->d_delta;
    if (shard_stride) *shard_stride = c->S;
    if (P64) *P64 = c->P64;
    return ACO_OK;
}

aco_status aco_gpu_set_pheromone(aco_gpu_ctx* c, const double* tau) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpy2DAsync(c->d_tau, c->P64 * sizeof(double), tau, c->n * sizeof(double),
                             c->n * sizeof(double), c->n, cudaMemcpyHostToDevice, c->stream));
        launch_rows(c, MODE_CHOICE);
        CK(cudaStreamSynchronize(c->stream));
    });
}

aco_status aco_gpu_compute_choice_info(aco_gpu_ctx* c) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        launch_rows(c, MODE_CHOICE);
        CK(cudaStreamSynchronize(c->stream));
    });
}

aco_status aco_gpu_construct(aco_gpu_ctx* c, aco_gpu_iter_record* rec) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        do_construct(c);
        if (c->sharded && !c->external) enqueue_shard_stats(c);
        CK(cudaMemcpyAsync(c->h_stats, c->d_stats, 8 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(c->h_stats + 8, c->d_fb, 3 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        aco_gpu_iter_record tmp{};
        aco_gpu_iter_record* r = rec ? rec : &tmp;
        const long long fb0 = c->h_stats[8], fb1 = c->h_stats[9];
        c->last_fb[0] = fb0;
        c->last_fb[1] = fb1;
        fill_common(c, r);
        finish_stats(c, r);
        r->construct_ms = ev_ms(c, 0, 2);
        r->construct_kernel_ms = ev_ms(c, 0, 1);
        r->fallbacks = fb0 + fb1;
        r->certified_fp64 = c->h_stats[10];
        r->best_so_far = c->best_so_far;
    });
}

aco_status aco_gpu_fold(aco_gpu_ctx* c, int32_t* row_blk) {
    if (c && !(c->external && c->row_shard)) {
        c->err = "aco_gpu_fold: the context does not row-shard its gather deposit "
                 "(needs external-exchange mode, world > 1, a gather deposit and rows of <= ~4000 doubles)";
        return ACO_E_CONFIG_ERROR;
    }
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        launch_rows(c, MODE_FOLD_OWN);
        CK(cudaStreamSynchronize(c->stream));
        c->folded = true;
        if (row_blk) *row_blk = c->row_blk;
    });
}

aco_status aco_gpu_update(aco_gpu_ctx* c, aco_gpu_iter_record* rec) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        do_update(c);
        CK(cudaStreamSynchronize(c->stream));
        if (rec) {
            rec->update_ms = ev_ms(c, 2, 5);
            rec->exchange_ms = ev_ms(c, 2, 3);
            rec->choice_ms = (!gather_mode(c) && !c->sharded) ? ev_ms(c, 4, 5) : 0.0;
        }
        ++c->iteration;
    });
}

aco_status aco_gpu_iterate(aco_gpu_ctx* c, aco_gpu_iter_record* rec, int32_t* tours_out,
                           int64_t* lengths_out) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        aco_gpu_iter_record tmp{};
        aco_gpu_iter_record* r = rec ? rec : &tmp;
        fill_common(c, r);
        // The one-warp-per-ant roulette streams each tour into a pinned,
        // device-mapped tours_out while it is built (32-entry chunks held in
        // the lanes, stored as each chunk closes); otherwise
        // the tours are copied after the construction.
        c->host_tours = nullptr;
        if (tours_out && c->cfg.selection == ACO_SEL_ROULETTE && !c->exact_only &&
            c->mloc > 0) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, tours_out) == cudaSuccess &&
                at.type == cudaMemoryTypeHost && at.devicePointer)
                c->host_tours = static_cast<int32_t*>(at.devicePointer);
            cudaGetLastError(); // pageable memory: not an error, just no mapping
        }
        const bool streamed = c->host_tours != nullptr;
        do_construct(c);
        c->host_tours = nullptr;
        // sharded: statistics and best tour reduced on the device, in stream
        // order before the update (no host round trip inside the iteration)
        if (c->sharded && !c->external) enqueue_shard_stats(c);
        // the tours are final once the construction phase (ev[2]) is done:
        // copy them out on a second stream while the update runs (the update
        // only reads them), and join before returning
        if (tours_out || lengths_out) {
            CK(cudaStreamWaitEvent(c->copy_stream, c->ev[2], 0));
            if (tours_out && !streamed)
                CK(cudaMemcpyAsync(tours_out, c->d_tours, sizeof(int32_t) * c->mloc * (c->n + 1),
                                   cudaMemcpyDeviceToHost, c->copy_stream));
            if (lengths_out)
                CK(cudaMemcpyAsync(lengths_out, c->d_len, sizeof(int64_t) * c->mloc,
                                   cudaMemcpyDeviceToHost, c->copy_stream));
        }
        do_update(c);
        CK(cudaMemcpyAsync(c->h_stats, c->d_stats, 8 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(c->h_stats + 8, c->d_fb, 3 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (tours_out || lengths_out) CK(cudaStreamSynchronize(c->copy_stream));
        finish_stats(c, r);
        r->construct_ms = ev_ms(c, 0, 2);
        r->construct_kernel_ms = ev_ms(c, 0, 1);
        r->update_ms = ev_ms(c, 2, 5);
        r->exchange_ms = ev_ms(c, 2, 3);
        r->choice_ms = (!gather_mode(c) && !c->sharded) ? ev_ms(c, 4, 5) : 0.0;
        r->fallbacks = c->h_stats[8] + c->h_stats[9];
        r->certified_fp64 = c->h_stats[10];
        c->last_fb[0] = c->h_stats[8];
        c->last_fb[1] = c->h_stats[9];
        r->best_so_far = c->best_so_far;
        ++c->iteration;
    });
}

aco_status aco_gpu_validate_tours(aco_gpu_ctx* c, const int32_t* tours, const int64_t* lengths,
                                  int32_t count) {
    return guard_ctx(c, [&] {
        if (count < 0 || (count > 0 && (!tours || !lengths)))
            throw ModelError(Errc::config_error, "tours and lengths are required");
        if (count == 0) return;
        CK(cudaSetDevice(c->device));
        int32_t* dt = nullptr;
        int64_t* dl = nullptr;
        const size_t tb = static_cast<size_t>(count) * (c->n + 1) * sizeof(int32_t);
        CK(cudaMalloc(&dt, tb));
        CK(cudaMalloc(&dl, count * sizeof(int64_t)));
        struct Free {
            void* a;
            void* b;
            ~Free() { cudaFree(a); cudaFree(b); }
        } guard{dt, dl};
        CK(cudaMemcpyAsync(dt, tours, tb, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(dl, lengths, count * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
        check_tours(c, dt, dl, count, 0);
    });
}

aco_status aco_gpu_get_pheromone(aco_gpu_ctx* c, double* tau) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpy2DAsync(tau, c->n * sizeof(double), c->d_tau, c->P64 * sizeof(double),
                             c->n * sizeof(double), c->n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

aco_status aco_gpu_get_choice(aco_gpu_ctx* c, double* choice) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaMemcpy2DAsync(choice, c->n * sizeof(double), c->d_choice, c->P64 * sizeof(double),
                             c->n * sizeof(double), c->n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

aco_status aco_gpu_get_topk(aco_gpu_ctx* c, int32_t* topk, int32_t* k) {
    return guard_ctx(c, [&] {
        if (!c->d_topk) throw Fail{ACO_E_UNSUPPORTED, "argmax cache not active"};
        CK(cudaSetDevice(c->device));
        if (k) *k = kTopK;
        if (topk)
            CK(cudaMemcpyAsync(topk, c->d_topk, static_cast<size_t>(c->n) * kTopK * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

aco_status aco_gpu_get_choice32(aco_gpu_ctx* c, float* choice, int32_t* scale_exp) {
    return guard_ctx(c, [&] {
        if (!c->d_choice32) throw Fail{ACO_E_UNSUPPORTED, "fp32 stream not active"};
        CK(cudaSetDevice(c->device));
        std::vector<float> raw(static_cast<size_t>(c->n) * c->PW);
        CK(cudaMemcpy(raw.data(), c->d_choice32, raw.size() * sizeof(float), cudaMemcpyDeviceToHost));
        if (scale_exp) CK(cudaMemcpy(scale_exp, c->d_scale, c->n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (int i = 0; i < c->n; ++i)
            for (int j = 0; j < c->n; ++j)
                choice[static_cast<size_t>(i) * c->n + j] =
                    raw[static_cast<size_t>(i) * c->PW + stream_pos(j, c->C, 4, c->LA, c->nat)];
    });
}

aco_status aco_gpu_get_tours(aco_gpu_ctx* c, int32_t* tours, int64_t* lengths) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        if (tours)
            CK(cudaMemcpyAsync(tours, c->d_tours, sizeof(int32_t) * c->mloc * (c->n + 1),
                               cudaMemcpyDeviceToHost, c->stream));
        if (lengths)
            CK(cudaMemcpyAsync(lengths, c->d_len, sizeof(int64_t) * c->mloc, cudaMemcpyDeviceToHost,
                               c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

aco_status aco_gpu_get_best(aco_gpu_ctx* c, int32_t* tour, int64_t* length) {
    return guard_ctx(c, [&] {
        CK(cudaSetDevice(c->device));
        if (tour)
            CK(cudaMemcpyAsync(tour, c->d_best, sizeof(int32_t) * (c->n + 1), cudaMemcpyDeviceToHost,
                               c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (length) *length = c->best_so_far;
    });
}

aco_status aco_gpu_get_info(aco_gpu_ctx* c, int32_t* m, int32_t* ant_begin, int32_t* ant_end,
                            double* tau0, int32_t* stream, int32_t* iteration) {
    if (!c) return ACO_E_CONFIG_ERROR;
    if (m) *m = c->m;
    if (ant_begin) *ant_begin = c->ant_begin;
    if (ant_end) *ant_end = c->ant_end;
    if (tau0) *tau0 = c->tau0;
    if (stream) *stream = c->stream_kind;
    if (iteration) *iteration = c->iteration;
    return ACO_OK;
}

aco_status aco_gpu_libm_pow(int32_t device, int32_t count, const double* xs, const double* ys,
                            double* out) {
    return guard_ctx(nullptr, [&] {
        CK(cudaSetDevice(device));
        LibmPowTables* tab = upload_pow_tables(nullptr);
        double *dx = nullptr, *dy = nullptr, *dout = nullptr;
        CK(cudaMalloc(&dx, count * sizeof(double)));
        CK(cudaMalloc(&dy, count * sizeof(double)));
        CK(cudaMalloc(&dout, count * sizeof(double)));
        CK(cudaMemcpy(dx, xs, count * sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dy, ys, count * sizeof(double), cudaMemcpyHostToDevice));
        k_libm_pow<<<std::max(1, std::min((count + 255) / 256, 4096)), 256>>>(dx, dy, count, tab, dout);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout, count * sizeof(double), cudaMemcpyDeviceToHost));
        cudaFree(dx);
        cudaFree(dy);
        cudaFree(dout);
        cudaFree(tab);
    });
}

aco_status aco_gpu_philox_uniform(int32_t device, uint64_t seed, uint32_t it, uint32_t ant,
                                  int32_t count, const uint32_t* steps, const uint32_t* draws,
                                  double* out) {
    return guard_ctx(nullptr, [&] {
        CK(cudaSetDevice(device));
        uint32_t *ds = nullptr, *dd = nullptr;
        double* dout = nullptr;
        CK(cudaMalloc(&ds, count * sizeof(uint32_t)));
        CK(cudaMalloc(&dd, count * sizeof(uint32_t)));
        CK(cudaMalloc(&dout, count * sizeof(double)));
        CK(cudaMemcpy(ds, steps, count * sizeof(uint32_t), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dd, draws, count * sizeof(uint32_t), cudaMemcpyHostToDevice));
        k_philox_test<<<(count + 255) / 256, 256>>>(seed, it, ant, count, ds, dd, dout);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, dout, count * sizeof(double), cudaMemcpyDeviceToHost));
        cudaFree(ds);
        cudaFree(dd);
        cudaFree(dout);
    });
}

} // extern "C"
