// Tour-construction kernels (sm_100a).
//
// Replaces the reference construction fork (engine.hpp:95-114) and its
// per-ant loop construct_tour (construction.hpp:181-201) with one WARP per
// ant.  Each of the n-1 dependent steps streams the current city's weight
// row from L2 with coalesced 128-bit loads, masks it with the ant's tabu
// bitmask (shared memory, construction.hpp:31-35 / model.hpp:88-114), and
// picks the next city.
//
// Roulette (select_next_roulette, construction.hpp:42-68).  The reference's
// choice is defined by SEQUENTIAL fp64 sums (total, then the walk), which a
// parallel reduction does not reproduce bit-for-bit.  The kernel therefore:
//   1. computes approximate prefix sums P_j (lane tree sums + warp scan),
//      with a rigorous error bound E against the exact real prefix X_j;
//   2. picks j* = first j with P_j > t = u * P_n;
//   3. CERTIFIES j*: if P_{j*} - t and t - P_{prev} both exceed
//      2 (E + E_ref + delta) (E_ref bounds the reference's own sequential
//      rounding, delta the rounding of its target u * total), the reference
//      provably returns j* (non-negative sums are monotone);
//   4. otherwise replays the reference arithmetic exactly (exact_walk): the
//      warp broadcasts the row 32 values at a time and every lane folds them
//      in ascending order, so the total, the target, the walk, last_positive
//      and the zero-total branch are the reference's own.
// The streamed row is either the fp64 choice (ACO_STREAM_FP64) or an fp32
// copy scaled per row by an exact power of two (ACO_STREAM_FP32); the fp32
// quantisation error (2^-24 relative + 2^-150 absolute) is part of E, and the
// exact walk always reads the fp64 choice, so both streams are bit-exact.
//
// Streamed layout ("lane-major within a round"): city c of round r lives at
//   r*32C + (t*32 + l)*V + q      with  c = r*32C + l*C + t*V + q,
// so the t-th 128-bit load of lane l (coalesced across the warp) returns
// cities l*C + tV .. +V-1: every lane owns a CONTIGUOUS chunk of C cities,
// which makes the in-order prefix a lane tree + one warp scan.
#pragma once

#include <cstdint>

#include "philox.cuh"

#ifndef ACO_SCAN_FMA
#define ACO_SCAN_FMA 1 // warp scan levels as shfl + fma (see warp_inclusive_scan); 0: shfl + predicated add + select
#endif
#ifndef ACO_TIMING
#define ACO_TIMING 0 // per-phase clock64() accounting into ConstructParams::timing
#endif

namespace acob200 {

constexpr unsigned kFull = 0xffffffffu;

template <typename WT> struct VecOf;
template <> struct VecOf<float> {
    using T = float4;
    static constexpr int V = 4;
};
template <> struct VecOf<double> {
    using T = double2;
    static constexpr int V = 2;
};

// Physical layout of a streamed row.  LA lanes share a row (32: one ant per
// warp; 16: two ants per warp), each owning C contiguous cities; a line of
// vectors has LA + 1 slots (one pad slot) so that reading one lane's chunk
// across a warp spreads over several bank groups.  Round r holds cities
// [r*LA*C, (r+1)*LA*C) in (LA+1)*C elements.
#ifndef ACO_PAD_SLOT
#define ACO_PAD_SLOT 1
#endif
constexpr int kPad = ACO_PAD_SLOT;
constexpr int kLP = 32 + kPad; // (LA + pad) for LA = 32

// Odd NV (vectors per lane chunk) may use the NATURAL layout instead (the
// context's `nat`: plain launches only — the relay launch measured slower
// with it, profiles/nat_layout_ab_r02.txt): city c at
// position c, lane l's vector t at slot l*NV + t.  Reading vector t of every
// lane strides the lanes NV (odd) slots apart, which spreads 32 lanes evenly
// over the 8 bank groups, and a lane's consecutive vectors sit in consecutive
// slots — conflict-free for both access patterns without a pad slot (pr2392:
// NV = 19, rows of 2432 floats instead of 2508).
template <int NV, bool NAT>
struct RowLayout {
    static constexpr bool nat = NAT && (NV & 1) != 0;
    static constexpr int lstr = nat ? NV : 1;               // vector stride between lanes
    static constexpr int tstr = nat ? 1 : kLP;              // between a lane's vectors
    static constexpr int round_vecs = nat ? 32 * NV : kLP * NV; // vectors per round
};

__host__ __device__ __forceinline__ int stream_pos(int c, int C, int V, int LA = 32, bool nat = false) {
    if (nat && ((C / V) & 1)) return c; // natural layout (odd NV)
    const int RC = LA * C, LP = LA + kPad;
    const int r = c / RC, rem = c - r * RC;
    const int l = rem / C, e = rem - l * C;
    const int t = e / V, q = e - t * V;
    return r * (LP * C) + (t * LP + l) * V + q;
}

// Inverse of stream_pos; returns INT_MAX for pad slots.
__host__ __device__ __forceinline__ int stream_city(int p, int C, int V, int LA = 32, bool nat = false) {
    if (nat && ((C / V) & 1)) return p; // natural layout (odd NV)
    const int LP = LA + kPad, RS = LP * C;
    const int r = p / RS, rem = p - r * RS;
    const int t = rem / (LP * V), rem2 = rem - t * LP * V;
    const int l = rem2 / V, q = rem2 - l * V;
    if (l >= LA) return 0x7fffffff;
    return r * LA * C + l * C + t * V + q;
}

#ifndef ACO_SEQ_GROUP
#define ACO_SEQ_GROUP 1 // high-occupancy roulette: predicated sequential group sums
#endif

#ifndef ACO_FUSED_TAIL_BUILD
#define ACO_FUSED_TAIL_BUILD 1 // 0: the kernels carry no tail (k_tour_length always runs)
#endif

struct ConstructParams {
    const void* w;           // streamed weights (float or double), row pitch PW
    const double* w64;       // natural fp64 choice, row pitch P64 (exact walk, nn)
    const int32_t* nn_lists; // n x nn (nn selection)
    const double* choice_nn; // n x nn weights of the nn lists (nn selection)
    const int2* choice_nn32;  // n x nn {city id, row-scaled fp32 weight bits} (nn <= 32) or null
    int32_t* tours;          // mloc x (n+1)
    unsigned long long* fallbacks;
    unsigned long long* argmax_fallbacks;
    unsigned long long* tier2; // roulette: steps certified by the fp64 re-sum (tier 2)
    int n, P64, PW, R, nn;
    int ant_begin, mloc;
    int random_start;
    int theta;
    int tabu_words; // per warp; >= PW/32 + 2
    uint32_t iteration;
    uint64_t seed;
    unsigned long long* timing; // ACO_TIMING: [8] phase cycle totals
    const int32_t* topk;        // nn selection: n x topk_k argmax cache (k_row_topk) or null
    int topk_k;
    int32_t* host_tours;        // device view of the caller's pinned tours_out (or null):
                                // the roulette kernel streams each tour there as it grows
    // fused tour tail (tour_tail, nn kernel): when len_out is set, the
    // construction kernel itself forms C_k and 1/C_k (and succ/pred when
    // set) and the separate k_tour_length launch is skipped.  (The roulette
    // kernel does not carry it: at 96 registers the extra code costs its
    // walk ~2.5%, more than the k_tour_length launch it would save.)
    const int32_t* dist;        // n x P64
    int64_t* len_out;           // mloc
    double* inv_out;            // this rank's block of [world][S]
    int32_t* succ_out;          // this rank's block of [world][n][S] (gather deposit) or null
    int32_t* pred_out;
    int S;
    // nn selection + accumulate deposit: per ant-step, the chosen city's
    // position in the current city's nn list (255: not a list member —
    // argmax fallback), so k_deposit_nn can fold list edges into the compact
    // n x nn slot array instead of scattering over n^2 tau
    uint8_t* qpos;              // mloc x n, or null
    // nn fast path (fp32 list weights, nn <= 32): its certification
    // constants, outward-rounded on the host (nn_certify_constants)
    float nn_e32, nn_lo32, nn_ce, nn_absq;
    // Relay (k_construct_roulette_relay): the grid is relay_W = SMs x q
    // warps, warp w owns ant w; the relay_E = mloc - relay_W leftover ants are
    // each built by relay_K warps in turn, one 32-aligned segment of steps
    // each (relay_bound), handing the tabu set and current city over through
    // global memory (relay_cur / relay_tabu) behind a release/acquire flag
    // stamped with relay_epoch.
    int relay_W, relay_E, relay_K;
    unsigned long long relay_epoch;
    unsigned long long* relay_flag; // [relay_E]
    int32_t* relay_cur;             // [relay_E]
    uint32_t* relay_tabu;           // [relay_E][tabu_words]
};

// First step of relay segment i of K over steps 1..n-1 (segment K ends at n);
// inner bounds are multiples of 32, so a segment's tour-stream chunks and
// Philox batches never straddle a hand-over (the host keeps (n-1)/K >= 33,
// so the 32-aligned bounds stay strictly increasing).
__host__ __device__ __forceinline__ int relay_bound(int i, int K, int n) {
    if (i <= 0) return 1;
    if (i >= K) return n;
    return static_cast<int>((static_cast<long long>(i) * (n - 1) / K) & ~31LL);
}

// Tour length (tour_length, model.hpp:205-226: an int64 sum, so any order is
// exact), w_k = 1.0 / (double)C_k (inverse_lengths, pheromone.hpp:123-128)
// and, for the row-gather deposit, the successor/predecessor tables — the
// same results k_tour_length forms, computed in the construction kernel's
// tail: the tour is read back from L2 right after it was built, eight edges
// per lane in flight, while the other warps on the SM are still walking.
// Plain loads for the tour (written by this kernel), __ldg for dist.
__device__ __forceinline__ void tour_tail(const ConstructParams& p, const int32_t* tour, int kl, int lane) {
    const int n = p.n;
    long long acc = 0;
    constexpr int B = 8;
    for (int s0 = lane; s0 < n; s0 += 32 * B) {
        int a[B], b[B], d[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int s = s0 + 32 * u;
            a[u] = s < n ? tour[s] : 0;
            b[u] = s < n ? tour[s + 1] : 0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u)
            d[u] = s0 + 32 * u < n ? __ldg(p.dist + static_cast<size_t>(a[u]) * p.P64 + b[u]) : 0;
        if (p.succ_out) {
#pragma unroll
            for (int u = 0; u < B; ++u)
                if (s0 + 32 * u < n) {
                    p.succ_out[static_cast<size_t>(a[u]) * p.S + kl] = b[u];
                    p.pred_out[static_cast<size_t>(b[u]) * p.S + kl] = a[u];
                }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) acc += d[u];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
    if (lane == 0) {
        p.len_out[kl] = acc;
        p.inv_out[kl] = 1.0 / static_cast<double>(acc);
    }
}

__device__ __forceinline__ bool tabu_test(const uint32_t* tabu, int j) {
    return (tabu[j >> 5] >> (j & 31)) & 1u;
}

// Lowest unvisited city (construction.hpp:31-35); pads >= n are preset.
__device__ __forceinline__ int lowest_unvisited(const uint32_t* tabu, int words, int lane) {
    for (int w0 = 0; w0 < words; w0 += 32) {
        const int wd = w0 + lane;
        const uint32_t free_bits = wd < words ? ~tabu[wd] : 0u;
        const unsigned b = __ballot_sync(kFull, free_bits != 0u);
        if (b) {
            const int src = __ffs(b) - 1;
            const uint32_t fb = __shfl_sync(kFull, free_bits, src);
            return (w0 + src) * 32 + __ffs(fb) - 1;
        }
    }
    return -1;
}

// Exact replay of select_next_roulette (construction.hpp:42-68) over the fp64
// row.  Every lane receives every weight by broadcast and folds them in
// ascending index order, so all lanes hold the reference's sequential sums.
// Visited cities contribute +0.0, which leaves a non-negative sum unchanged
// and can never trigger "acc > target" or last_positive, exactly like the
// reference's `continue`.  The running sum at every 32-city boundary is kept
// in `chunk_start` (shared, >= ceil(n/32) doubles), so after the total is
// known only the crossing chunk is re-folded — from its stored start value,
// which reproduces the same sequential sums bit for bit.
// TMA / mbarrier helpers (cp.async.bulk 1-D copies into shared memory).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// The fp64 row is staged through the shared row buffer (`stage`, stage_bytes
// >= 256) in pieces with TMA, and every lane folds every weight from
// broadcast shared loads (same address in all lanes), so the only dependence
// chain is the reference's own sequential fp64 add.
// Number of staging pieces (mbarrier phases) one exact_walk consumes; the
// caller advances its phase by this parity (phase is passed by value so it
// stays in a register in the hot loop).
__host__ __device__ __forceinline__ int exact_walk_pieces(int n, uint32_t stage_bytes) {
    const int piece = static_cast<int>(stage_bytes / 256) * 32;
    return (n + piece - 1) / piece;
}

__device__ __noinline__ int exact_walk(const double* __restrict__ row, const uint32_t* tabu,
                                       int n, int words, double u, int lane,
                                       double* chunk_start, double* stage, uint32_t stage_bytes,
                                       uint64_t* bar, uint32_t phase) {
    const int nch = (n + 31) >> 5;
    const int piece = static_cast<int>(stage_bytes / 256) * 32; // cities per piece (chunk-aligned)
    double acc = 0.0;
    int last_positive = -1;
    for (int p0 = 0; p0 < n; p0 += piece) {
        const int cnt = min(piece, n - p0);
        const uint32_t bytes = static_cast<uint32_t>(((cnt * 8) + 15) & ~15);
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async_smem();
            mbar_expect_tx(bar, bytes);
            tma_row(stage, row + p0, bytes, bar);
        }
        __syncwarp();
        mbar_wait(bar, phase);
        phase ^= 1u;
        for (int c = p0 >> 5; c < ((p0 + cnt + 31) >> 5); ++c) {
            const int base = c << 5;
            const uint32_t vis = tabu[c];
            const double2* s2 = reinterpret_cast<const double2*>(stage + (base - p0));
            if (lane == 0) chunk_start[c] = acc;
            unsigned pos = 0;
#pragma unroll
            for (int q2 = 0; q2 < 16; ++q2) {
                double2 v = make_double2(0.0, 0.0);
                if (base + 2 * q2 < n) v = s2[q2];
                const double x0 = ((vis >> (2 * q2)) & 1u) ? 0.0 : v.x;
                const double x1 = ((vis >> (2 * q2 + 1)) & 1u) ? 0.0 : v.y;
                pos |= (x0 > 0.0 ? 1u : 0u) << (2 * q2);
                pos |= (x1 > 0.0 ? 1u : 0u) << (2 * q2 + 1);
                acc += x0;
                acc += x1;
            }
            if (pos) last_positive = base + 31 - __clz(pos);
        }
    }
    __syncwarp();
    if (!(acc > 0.0)) return lowest_unvisited(tabu, words, lane); // total <= 0 (:52)
    const double target = u * acc;                                  // :54
    // the crossing lies in the first chunk whose end sum exceeds the target
    int ch = -1;
    for (int c0 = 0; c0 < nch && ch < 0; c0 += 32) {
        const int c = c0 + lane;
        const double end = c < nch ? (c + 1 < nch ? chunk_start[c + 1] : acc) : -1.0;
        const unsigned b = __ballot_sync(kFull, c < nch && end > target);
        if (b) ch = c0 + __ffs(b) - 1;
    }
    if (ch < 0) return last_positive >= 0 ? last_positive : lowest_unvisited(tabu, words, lane);
    // re-fold the crossing chunk from its stored start: lane q keeps the sum
    // after city base+q (the same sequential adds, so the same values)
    const int base = ch << 5;
    const int j = base + lane;
    const double w = (j < n && !tabu_test(tabu, j)) ? __ldg(row + j) : 0.0;
    double a2 = chunk_start[ch], mine = 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
        a2 += __shfl_sync(kFull, w, q);
        mine = (q == lane) ? a2 : mine;
    }
    const unsigned cross = __ballot_sync(kFull, mine > target);
    return base + __ffs(cross) - 1; // first prefix > target (:62)
}

template <typename WT, int C>
__device__ __forceinline__ WT tree_sum(WT (&x)[C]) {
#pragma unroll
    for (int s = 1; s < C; s <<= 1) {
#pragma unroll
        for (int i = 0; i + s < C; i += 2 * s) x[i] += x[i + s];
    }
    return x[0];
}

// Packed (f32x2, sm_100 FADD2) pairwise tree over an even-length group:
// depth ceil(log2(N)), the same error bound as the scalar tree.
template <int N>
__device__ __forceinline__ float tree_sum_packed(float (&x)[N]) {
    static_assert(N % 2 == 0, "even group");
    float2 y[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) y[i] = make_float2(x[i], x[N / 2 + i]);
#pragma unroll
    for (int s = 1; s < N / 2; s <<= 1) {
#pragma unroll
        for (int i = 0; i + s < N / 2; i += 2 * s) y[i] = __fadd2_rn(y[i], y[i + s]);
    }
    return y[0].x + y[0].y;
}

// Inclusive warp scan step without a lane-index compare: shfl.sync.up's
// predicate output says whether the source lane existed.
__device__ __forceinline__ float scan_up_add(float v, int off) {
    float y;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "shfl.sync.up.b32 %0|p, %1, %2, 0, -1;\n\t"
        "@p add.rn.f32 %0, %0, %1;\n\t"
        "@!p mov.b32 %0, %1;\n}"
        : "=f"(y)
        : "f"(v), "r"(off));
    return y;
}
// in-place form: the source-lane predicate of shfl.up guards an add into v
// itself — two dependent instructions per level, no select, no mask registers
__device__ __forceinline__ void scan_up_add_inplace(float& v, int off) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .f32 y;\n\t"
        "shfl.sync.up.b32 y|p, %0, %1, 0, -1;\n\t"
        "@p add.rn.f32 %0, %0, y;\n}"
        : "+f"(v)
        : "r"(off));
}
// INPLACE: the predicated in-place form (fewer instructions: pays at high
// occupancy, where issue slots are scarce; the fma form's shorter chain pays
// in latency-bound launches)
template <bool INPLACE = false>
__device__ __forceinline__ float warp_inclusive_scan(float v) {
    if constexpr (INPLACE) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) scan_up_add_inplace(v, off);
        return v;
    }
#if ACO_SCAN_FMA
    // two dependent instructions per level instead of three: with m = 1 for
    // lanes >= off (else 0), fma(y, m, v) is fl(v + y) or exactly v — the
    // same values as scan_up_add for the finite non-negative sums scanned
    // here (0 * y = +0 needs y finite)
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float y = __shfl_up_sync(kFull, v, off);
        v = __fmaf_rn(y, lane >= off ? 1.f : 0.f, v);
    }
#else
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = scan_up_add(v, off);
#endif
    return v;
}

template <int C>
__host__ __device__ constexpr int ceil_log2() {
    int d = 0;
    while ((1 << d) < C) ++d;
    return d;
}

__device__ __forceinline__ void tabu_init(uint32_t* tabu, int words, int n, int lane) {
    for (int wd = lane; wd < words; wd += 32) {
        const int c0 = wd * 32;
        uint32_t v;
        if (c0 + 32 <= n) v = 0u;
        else if (c0 >= n) v = kFull;
        else v = kFull << (n - c0);
        tabu[wd] = v;
    }
}

__device__ __forceinline__ int start_city(const ConstructParams& p, uint32_t kg) {
    if (p.random_start) { // engine.hpp:105-108: burns draw 0 of step 0
        int s = static_cast<int>(philox_uniform(p.seed, p.iteration, kg, 0, 0) * p.n);
        return s >= p.n ? p.n - 1 : s;
    }
    return static_cast<int>(kg % static_cast<uint32_t>(p.n));
}

// ---------------------------------------------------------------------------
// Middle certification tier: the streamed (fp32) row is still in shared
// memory; redo every prefix sum in fp64 from it.  The only approximation left
// is the fp32 quantisation of the weights (2^-24 relative + 2^-150 absolute per
// city), so the uncertainty band is ~15x narrower than the fp32 pass's.
// Returns the certified city or -1.
template <typename WT, int NV, int MAXR, bool NAT = false>
__device__ __noinline__ int certify_fp64(const WT* buf, const uint32_t* tabu, int n, int R,
                                          double u, int lane) {
    using VT = typename VecOf<WT>::T;
    constexpr int V = VecOf<WT>::V;
    constexpr int C = NV * V;
    constexpr int NWIN = (C + 31) / 32;
    constexpr bool F32 = sizeof(WT) == 4;
    const double e_rel = ((F32 ? 2.0 * 0x1.0p-24 : 0.0) +
                          (double)(2 * C + MAXR + 16) * 0x1.0p-53 +
                          (double)(n + 8) * 0x1.0p-53) * (1.0 + 0x1.0p-16);
    const double abs_q = F32 ? (double)n * 0x1.0p-149 : 0.0;
    double lsum[MAXR];
    double incl[MAXR];
    double T = 0.0;
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
        lsum[r] = 0.0;
        incl[r] = 0.0;
        if (r < R) {
            const int cbase = r * 32 * C + lane * C;
            const int w0 = cbase >> 5, sh = cbase & 31;
            uint32_t win[NWIN];
#pragma unroll
            for (int i = 0; i < NWIN; ++i) win[i] = __funnelshift_r(tabu[w0 + i], tabu[w0 + i + 1], sh);
            const VT* rv = reinterpret_cast<const VT*>(buf + r * RowLayout<NV, NAT>::round_vecs * V) +
                           lane * RowLayout<NV, NAT>::lstr;
            double acc = 0.0;
#pragma unroll
            for (int tv = 0; tv < NV; ++tv) {
                const VT v = rv[tv * RowLayout<NV, NAT>::tstr];
                WT xs[V];
                if constexpr (F32) { xs[0] = v.x; xs[1] = v.y; xs[2] = v.z; xs[3] = v.w; }
                else { xs[0] = v.x; xs[1] = v.y; }
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    const int e = tv * V + q;
                    if (!((win[e >> 5] >> (e & 31)) & 1u)) acc += static_cast<double>(xs[q]);
                }
            }
            lsum[r] = acc;
            double d = acc;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const double y = __shfl_up_sync(kFull, d, off);
                if (lane >= off) d += y;
            }
            incl[r] = d;
            T += __shfl_sync(kFull, d, 31);
        }
    }
    if (!(T > 0.0) || !(T < 1e300)) return -1;
    const double t = u * T;
    double base = 0.0, my = 0.0, mys = 0.0;
    int rs = -1;
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
        if (r < R && rs < 0) {
            const double rt = __shfl_sync(kFull, incl[r], 31);
            if (base + rt > t) {
                rs = r;
                my = incl[r];
                mys = lsum[r];
            } else {
                base += rt;
            }
        }
    }
    if (rs < 0) return -1;
    const unsigned bal = __ballot_sync(kFull, base + my > t);
    if (!bal) return -1;
    const int L = __ffs(bal) - 1;
    int J = -1;
    bool cert = false;
    if (lane == L) {
        double acc = base + (my - mys);
        const int cbase = rs * 32 * C + L * C;
        const WT* chunk = buf + rs * RowLayout<NV, NAT>::round_vecs * V;
        for (int e = 0; e < C; ++e) {
            const int c = cbase + e;
            if (tabu_test(tabu, c)) continue;
            const double x = static_cast<double>(chunk[((e / V) * RowLayout<NV, NAT>::tstr + L * RowLayout<NV, NAT>::lstr) * V + (e % V)]);
            const double na = acc + x;
            if (x > 0.0 && na > t) {
                const double Thi = T * (1.0 + 0x1.0p-16) + abs_q;
                const double Mt = (e_rel + 0x1.0p-50) * (u * Thi) + abs_q;
                cert = (na * (1.0 - e_rel) - 2.0 * abs_q > t + Mt) &&
                       (acc + e_rel * na + 2.0 * abs_q < t - Mt);
                J = c;
                break;
            }
            acc = na;
        }
    }
    J = __shfl_sync(kFull, J, L);
    const bool c2 = __shfl_sync(kFull, cert, L);
    return (c2 && J >= 0 && J < n) ? J : -1;
}

// ---------------------------------------------------------------------------
// Roulette over the full row, one warp (= one CTA) per ant.  Per step:
//   1. the row (PW * sizeof(WT) bytes) is in shared memory: one cp.async.bulk
//      (TMA) per step, issued SPECULATIVELY for the likely next city as soon
//      as j* is located, so the L2 latency overlaps certification and
//      bookkeeping (if certification fails the copy is drained and the true
//      row fetched);
//   2. lane l reads its contiguous chunk (NV conflict-free 128-bit LDS),
//      masks it with its tabu window and tree-sums it in groups of GE cities;
//      one warp scan of the lane sums gives T and t = u*T;
//   3. every lane walks its OWN chunk branch-free: group prefix (NG adds) ->
//      Kogge-Stone prefix of the GE cities of the crossing group -> compare
//      bitmask -> ffs; each lane certifies its own candidate, so selecting
//      the result is two ballots and one shuffle.
// All of 2-3 run in the accumulation type AT: fp32 for the fp32 stream (the
// fp32 adds on any prefix path are counted in the bound, ~24 * 2^-24), fp64
// for the fp64 stream.  Only the final two certification compares are fp64.
// NV = 128-bit vectors per lane per round, C = NV*V, MAXR = max rounds.
// One ant in the roulette kernels: the state a run of steps carries.
struct RouletteAnt {
    int kl;           // local ant index (tour row)
    uint32_t kg;      // global ant id (RNG key)
    int32_t* tour;
    uint32_t* tabu;   // shared-memory tabu bitmask
    int cur;          // current city
    bool prefetched;  // the row of `cur` is already requested (speculative TMA)
};

// Lays the ant's start city down (tabu, tour[0]).
__device__ __forceinline__ void roulette_begin(const ConstructParams& p, RouletteAnt& a, int kl,
                                               uint32_t* tabu, int lane, bool stream) {
    a.kl = kl;
    a.kg = static_cast<uint32_t>(p.ant_begin + kl);
    a.tour = p.tours + static_cast<size_t>(kl) * (p.n + 1);
    a.tabu = tabu;
    a.prefetched = false;
    tabu_init(tabu, p.tabu_words, p.n, lane);
    const int start = start_city(p, a.kg);
    __syncwarp();
    if (lane == 0) {
        tabu[start >> 5] |= 1u << (start & 31);
        a.tour[0] = start;
    }
    if (stream && lane == 0) p.host_tours[static_cast<size_t>(kl) * (p.n + 1)] = start; // mapped tours_out
    a.cur = start;
}

// Closes the tour (tour[n] = start).
__device__ __forceinline__ void roulette_end(const ConstructParams& p, RouletteAnt& a, int lane, bool stream) {
    const int start = start_city(p, a.kg);
    if (lane == 0) {
        a.tour[p.n] = start;
        if (stream) p.host_tours[static_cast<size_t>(a.kl) * (p.n + 1) + p.n] = start;
    }
    __syncwarp();
}

// Steps [s0, s1) of one ant.  smem: the kernel's dynamic shared memory
// (mbarrier, row buffer, own tabu, chunk_start, gsum).
template <typename WT, int NV, int MAXR, bool STREAM, bool SCAN_INPLACE = false, bool SEQG = false,
          bool NAT = false>
__device__ __forceinline__ void roulette_steps(const ConstructParams& p, RouletteAnt& a, int s0, int s1,
                                               unsigned char* smem_raw, uint32_t& phase,
                                               unsigned long long& fb, unsigned long long& fb2) {
    using VT = typename VecOf<WT>::T;
    using AT = WT; // accumulation type
    constexpr int V = VecOf<WT>::V;
    constexpr int C = NV * V;
    constexpr int NWIN = (C + 31) / 32;
    constexpr int GV = 4;                              // vectors per tree group
    constexpr int NG = (NV + GV - 1) / GV;             // groups per chunk
    constexpr int GE = GV * V;                         // cities per group
    constexpr bool F32 = sizeof(WT) == 4;
    using RL = RowLayout<NV, NAT>;
    // SEQ: high-occupancy launches (SEQG) sum each group of GE
    // cities with predicated sequential adds (GE instructions, no masking
    // selects) instead of masked selects + a packed tree (GE + GE/2): fewer
    // issue slots, a longer chain (hidden by the other warps there)
    constexpr bool SEQ = ACO_SEQ_GROUP && SEQG && F32 && MAXR == 1;
    constexpr int D1 = (SEQ ? GE - 1 : ceil_log2<GE>()) + ceil_log2<NG>();
    // fp32 single-round rows: the group walk; otherwise the quad-scan walk
    constexpr bool kGroupWalk = F32 && MAXR == 1;
    static_assert(GE <= 32 && 32 % GE == 0, "a group's bits live in one window word");

    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    WT* buf = reinterpret_cast<WT*>(smem_raw + 128);
    double* chunk_start = reinterpret_cast<double*>(
        reinterpret_cast<uint32_t*>(smem_raw + 128 + static_cast<size_t>(p.PW) * sizeof(WT)) + p.tabu_words);
    WT* gsum = reinterpret_cast<WT*>(chunk_start + ((p.n + 31) >> 5)); // [MAXR][NG][32]
    const int lane = threadIdx.x & 31;
    const int n = p.n;
    const WT* __restrict__ wbase = static_cast<const WT*>(p.w);
    const uint32_t row_bytes = static_cast<uint32_t>(p.PW * sizeof(WT));

    // e: bound on |P_j - X_j| / X_j for every prefix estimate (AT adds along
    // any path: tree D1, warp scan 5, round bases MAXR, group prefix NG,
    // Kogge-Stone log2 GE, 3 more; + fp32 quantisation of the summands and of
    // x_j* in Pprev) plus the reference's own sequential error gamma_n.
    constexpr double ulp_at = F32 ? 0x1.0p-24 : 0x1.0p-53;
    const double e_rel =
        ((double)(D1 + 5 + MAXR + 1 + 2 + 5 + 4 + 3) * ulp_at +
         (F32 ? 2.0 * 0x1.0p-24 : 0.0) + (double)(n + 8) * 0x1.0p-53) * (1.0 + 0x1.0p-16);
    const double abs_q = F32 ? (double)n * 0x1.0p-149 : 0.0;
    const double lo_f = 1.0 - e_rel;
    const float lo32 = __double2float_rd(lo_f); // <= lo_f
    const float e32 = __double2float_ru(e_rel); // >= e_rel
    const float ce32 = __double2float_ru(e_rel + 4.0 * ulp_at); // >= the Mt coefficient
    const float absq32 = __double2float_ru(abs_q);              // n * 2^-149 (exact)

    const int kl = a.kl;
    const uint32_t kg = a.kg;
    int32_t* const tour = a.tour;
    uint32_t* const tabu = a.tabu;
    int cur = a.cur;
    bool prefetched = a.prefetched;
    // STREAM: lane (s & 31) holds tour[s] of the open 32-entry chunk; the
    // chunk is stored when it closes (or the run ends), to the device tour
    // and to the caller's mapped pinned tours_out alike — one coalesced
    // 128-byte write each, no per-step store and no read-back.  (Without a
    // host buffer lane 0 stores every step: measured no slower there.)
    int held = 0;
    // Draw 0 of steps b..b+31 (b = 1 mod 32): lane i holds step b + i
    // (rng.hpp:74-80); a run starting inside a batch draws it first.
    double ubatch = 0.0;
    float ub_dn = 0.f, ub_up = 0.f; // kGroupWalk: the draw rounded down / up
    if (((s0 - 1) & 31) != 0) {
        ubatch = philox_uniform(p.seed, p.iteration, kg, static_cast<uint32_t>(((s0 - 1) & ~31) + 1 + lane), 0);
        ub_dn = __double2float_rd(ubatch);
        ub_up = __double2float_ru(ubatch);
    }
#if ACO_TIMING
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tk = clock64();
#define TICK(i) do { const long long t_ = clock64(); ph[i] += t_ - tk; tk = t_; } while (0)
#else
#define TICK(i) do {} while (0)
#endif

    for (int step = s0; step < s1; ++step) {
        if (!prefetched && lane == 0) { // (normally the previous step requested this row)
            fence_proxy_async_smem(); // generic reads of buf happen-before the refill
            mbar_expect_tx(bar, row_bytes);
            tma_row(buf, wbase + static_cast<size_t>(cur) * p.PW, row_bytes, bar);
        }
        // Draw 0 of steps step..step+31: lane i holds step + i (rng.hpp:74-80).
        if (((step - 1) & 31) == 0) {
            ubatch = philox_uniform(p.seed, p.iteration, kg,
                                    static_cast<uint32_t>(step + lane), 0);
            if constexpr (kGroupWalk) {
                ub_dn = __double2float_rd(ubatch);
                ub_up = __double2float_ru(ubatch);
            }
        }
        // the group walk brackets u by the float pair (u_dn <= u <= u_up):
        // candidate and certification thresholds in fp32, no conversions;
        // the fp64 draw is shuffled only when a fallback tier runs
        double u = 0.0;
        float u32 = 0.f, u_dn = 0.f, u_up = 0.f;
        if constexpr (kGroupWalk) {
            u_dn = __shfl_sync(kFull, ub_dn, (step - 1) & 31);
            u_up = __shfl_sync(kFull, ub_up, (step - 1) & 31);
        } else {
            u = __shfl_sync(kFull, ubatch, (step - 1) & 31);
            u32 = __double2float_rn(u);
        }
        __syncwarp();
        mbar_wait(bar, phase);
        phase ^= 1u;
        prefetched = false;
        const WT* rowsrc = buf; // the staged row
        TICK(6);

        AT incl[MAXR];
        AT rtot[MAXR];
        WT gsr[NG]; // MAXR == 1: lane-local inclusive prefix of the group sums
        AT T = AT(0);
#pragma unroll
        for (int r = 0; r < MAXR; ++r) {
            incl[r] = AT(0);
            rtot[r] = AT(0);
            if (MAXR == 1 || r < p.R) { // single-round layouts have R == 1
                const int cbase = r * 32 * C + lane * C;
                const int w0 = cbase >> 5, sh = cbase & 31;
                uint32_t win[NWIN];
#pragma unroll
                for (int i = 0; i < NWIN; ++i)
                    win[i] = __funnelshift_r(tabu[w0 + i], tabu[w0 + i + 1], sh);
                const VT* rv = reinterpret_cast<const VT*>(rowsrc + r * RL::round_vecs * V) + lane * RL::lstr;
                WT gs[NG];
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    WT x[GE];
#pragma unroll
                    for (int tt = 0; tt < GV; ++tt) {
                        const int tv = g * GV + tt;
                        VT v;
                        if (tv < NV) {
                            v = rv[tv * RL::tstr];
                        } else {
                            if constexpr (F32) v = make_float4(0.f, 0.f, 0.f, 0.f);
                            else v = make_double2(0.0, 0.0);
                        }
                        if constexpr (F32) {
                            x[tt * 4 + 0] = v.x; x[tt * 4 + 1] = v.y;
                            x[tt * 4 + 2] = v.z; x[tt * 4 + 3] = v.w;
                        } else {
                            x[tt * 2 + 0] = v.x; x[tt * 2 + 1] = v.y;
                        }
                    }
                    if constexpr (SEQ) {
                        WT acc = WT(0);
#pragma unroll
                        for (int e = 0; e < GE; ++e) {
                            const int ee = g * GE + e;
                            if (ee < C && !((win[ee >> 5] >> (ee & 31)) & 1u)) acc += x[e];
                        }
                        gs[g] = acc;
                    } else {
#pragma unroll
                    for (int e = 0; e < GE; ++e) {
                        const int ee = g * GE + e;
                        if (ee < C && ((win[ee >> 5] >> (ee & 31)) & 1u)) x[e] = WT(0);
                    }
                    if constexpr (F32) gs[g] = tree_sum_packed<GE>(x);
                    else gs[g] = tree_sum<WT, GE>(x);
                    }
                    if constexpr (MAXR > 1) gsum[(r * NG + g) * 32 + lane] = gs[g];
                }
                if constexpr (MAXR == 1) { // lane-local inclusive group prefixes
                    gsr[0] = gs[0];
#pragma unroll
                    for (int g = 1; g < NG; ++g) gsr[g] = gsr[g - 1] + gs[g];
                }
                AT d = static_cast<AT>(tree_sum<WT, NG>(gs));
                TICK(0);
                if constexpr (F32) {
                    d = warp_inclusive_scan<SCAN_INPLACE>(d);
                } else {
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const AT y = __shfl_up_sync(kFull, d, off);
                        if (lane >= off) d += y;
                    }
                }
                incl[r] = d;
                rtot[r] = __shfl_sync(kFull, d, 31);
                T += rtot[r];
                TICK(1);
            }
        }
        const double Td = static_cast<double>(T);
        const double tdd = u * Td;
        // Candidate threshold in AT.  Only the candidate search uses it —
        // certification compares against tdd through A and B — so the
        // fp32 stream forms it in fp32 from a float copy of u (known at
        // the top of the step), keeping the double product and its two
        // conversions off the scan -> ballot chain.
        AT t;
        if constexpr (kGroupWalk) t = __fmul_rn(u_dn, T);
        else if constexpr (F32) t = __fmul_rn(u32, T);
        else t = static_cast<AT>(tdd);
        // certification thresholds (T, u only): |t_ref - t| <= Mt
        const double Thi = Td * (1.0 + 0x1.0p-16) + abs_q;
        const double Mt = (e_rel + 4.0 * ulp_at) * (u * Thi) + abs_q; // + rounding of t to AT
        const double A = tdd + Mt + 2.0 * abs_q; // need Pj * (1 - e) > A
        const double B = tdd - Mt - 2.0 * abs_q; // need Pprev + e * Pj < B
        // the group walk's fp32 form, every operation rounded outward:
        // A32 >= u*T + Mt + 2*abs >= A's real value, B32 <= u*T - Mt - 2*abs
        float A32 = 0.f, B32 = 0.f;
        if constexpr (kGroupWalk) {
            const float Thi32 = __fadd_ru(__fmul_ru(T, 1.0f + 0x1.0p-16f), absq32);
            const float Mt32 = __fadd_ru(__fmul_ru(ce32, __fmul_ru(u_up, Thi32)), absq32);
            A32 = __fadd_ru(__fadd_ru(__fmul_ru(u_up, T), Mt32), 2.0f * absq32);
            B32 = __fsub_rd(__fsub_rd(__fmul_rd(u_dn, T), Mt32), 2.0f * absq32);
        }
        bool ok;
        if constexpr (kGroupWalk) ok = (T > AT(0)) && (T <= 0x1.fffffep127f);
        else ok = (T > AT(0)) && (Td < 1e300);
        int next = -1;
        if (ok) {
            AT base = AT(0), my = AT(0);
            int rs = -1;
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                if ((MAXR == 1 || r < p.R) && rs < 0) {
                    if (base + rtot[r] > t) {
                        rs = r;
                        my = incl[r];
                    } else {
                        base += rtot[r];
                    }
                }
            }
            int J = -1;        // candidate city (global index), valid in lane Q
            bool cert = false; // its certification
            if constexpr (kGroupWalk) {
                // Group walk (MAXR == 1, fp32): every lane locates the
                // crossing GROUP of its own chunk from its group prefixes
                // (no extra shared reads); lane L's group G and exclusive
                // base are broadcast, and lanes 0..3 each take one 4-city
                // quad of that group: quad prefixes by three parallel
                // shuffles, the first crossing city by one ballot.
                const AT exo = __shfl_up_sync(kFull, incl[0], 1);
                const AT excl_own = lane == 0 ? AT(0) : exo;
                const unsigned lb = __ballot_sync(kFull, incl[0] > t);
                // crossing group of the own chunk: the number of group
                // prefixes <= t - excl_own (a wrong pick in a rounding tie
                // only fails certification); its exclusive base.
                const AT tl = t - excl_own;
                int Gown = 0;
                AT gb = AT(0);
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    const bool below = gsr[g] <= tl;
                    Gown += below ? 1 : 0;
                    gb = below ? gsr[g] : gb;
                }
                const AT bG = excl_own + gb;
                if (lb) {
                    const int L = __ffs(lb) - 1;
                    const int G = __shfl_sync(kFull, Gown, L);
                    const AT baseG = __shfl_sync(kFull, bG, L);
                    if (G < NG) {
                        const int k = lane & 3;
                        const int tv = G * GV + k;
                        const int c0 = L * C + tv * 4; // first city of the quad
                        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                        uint32_t bits4 = 0xFu;
                        if (tv < NV) {
                            v = reinterpret_cast<const float4*>(buf)[tv * RL::tstr + L * RL::lstr];
                            bits4 = __funnelshift_r(tabu[c0 >> 5], tabu[(c0 >> 5) + 1], c0 & 31);
                        }
                        AT x0 = (bits4 & 1u) ? AT(0) : v.x;
                        AT x1 = (bits4 & 2u) ? AT(0) : v.y;
                        AT x2 = (bits4 & 4u) ? AT(0) : v.z;
                        AT x3 = (bits4 & 8u) ? AT(0) : v.w;
                        const AT a1 = x0 + x1;
                        const AT a2 = a1 + x2;
                        const AT a3 = a2 + x3;
                        const AT s1 = __shfl_up_sync(kFull, a3, 1, 4);
                        const AT s2 = __shfl_up_sync(kFull, a3, 2, 4);
                        const AT s3 = __shfl_up_sync(kFull, a3, 3, 4);
                        const AT ex = (k >= 1 ? s1 : AT(0)) + ((k >= 2 ? s2 : AT(0)) + (k >= 3 ? s3 : AT(0)));
                        const AT kb = baseG + ex;
                        const AT p0 = kb + x0, p1 = kb + a1, p2 = kb + a2, p3 = kb + a3;
                        int E = -1;
                        AT Pj32 = AT(0), Pp32 = AT(0);
                        // first q with x_q > 0 and P_q > t (descending so the lowest wins)
                        if (x3 > AT(0) && p3 > t) { E = 3; Pj32 = p3; Pp32 = p2; }
                        if (x2 > AT(0) && p2 > t) { E = 2; Pj32 = p2; Pp32 = p1; }
                        if (x1 > AT(0) && p1 > t) { E = 1; Pj32 = p1; Pp32 = p0; }
                        if (x0 > AT(0) && p0 > t) { E = 0; Pj32 = p0; Pp32 = kb; }
                        const unsigned qb = __ballot_sync(kFull, lane < 4 && E >= 0);
                        const bool mine = qb != 0u && lane == __ffs(qb) - 1;
                        // The certification in fp32 with directed rounding
                        // (implies the fp64 form): Pj*lo_f >= rd(Pj*lo32) >
                        // A32 >= A and Pprev + e*Pj <= ru(Pprev + ru(e32*Pj))
                        // < B32 <= B, with lo32 <= lo_f, e32 >= e_rel.
                        const int Jc = c0 + E;
                        J = mine ? Jc : -1;
                        cert = mine && (__fmul_rd(Pj32, lo32) > A32) &&
                               (__fadd_ru(Pp32, __fmul_ru(e32, Pj32)) < B32) && Jc < n;
                    }
                }
            } else {
                // crossing lane L of round rs, then a cooperative walk over L's
                // chunk: lane k takes quad k (4 consecutive cities), quad sums are
                // scanned across the warp, and the lane holding the crossing quad
                // walks its 4 cities.
                const unsigned lb = __ballot_sync(kFull, rs >= 0 && base + my > t);
                int Q = -1;
                if (lb) {
                    const int L = __ffs(lb) - 1;
                    const AT myprev = __shfl_sync(kFull, my, L == 0 ? 0 : L - 1);
                    const AT exclL = base + (L == 0 ? AT(0) : myprev);
                    constexpr int NQT = C / 4; // quads per chunk
                    const int cbaseL = rs * 32 * C + L * C;
                    // all lanes load (lanes >= NQT re-read quad 0 and drop it)
                    const int ql = lane < NQT ? lane : 0;
                    AT xv[4];
                    if constexpr (F32) {
                        const float4* qp = reinterpret_cast<const float4*>(
                            rowsrc + rs * RL::round_vecs * V + (ql * RL::tstr + L * RL::lstr) * 4);
                        const float4 v = *qp;
                        xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
                    } else {
                        const double2 v0 = *reinterpret_cast<const double2*>(
                            buf + rs * RL::round_vecs * V + ((2 * ql) * RL::tstr + L * RL::lstr) * 2);
                        const double2 v1 = *reinterpret_cast<const double2*>(
                            buf + rs * RL::round_vecs * V + ((2 * ql + 1) * RL::tstr + L * RL::lstr) * 2);
                        xv[0] = v0.x; xv[1] = v0.y; xv[2] = v1.x; xv[3] = v1.y;
                    }
                    {
                        const int c0 = cbaseL + 4 * ql;
                        uint32_t bits4 =
                            __funnelshift_r(tabu[c0 >> 5], tabu[(c0 >> 5) + 1], c0 & 31);
                        if (lane >= NQT) bits4 = 0xFu;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if ((bits4 >> q) & 1u) xv[q] = AT(0);
                    }
                    const AT qs = (xv[0] + xv[1]) + (xv[2] + xv[3]);
                    AT qi = qs;
                    if constexpr (F32) {
                        qi = warp_inclusive_scan(qi);
                    } else {
#pragma unroll
                        for (int off = 1; off < 32; off <<= 1) {
                            const AT y = __shfl_up_sync(kFull, qi, off);
                            if (lane >= off) qi += y;
                        }
                    }
                    const AT qe = __shfl_up_sync(kFull, qi, 1);
                    const unsigned qb = __ballot_sync(kFull, lane < NQT && exclL + qi > t);
                    Q = __ffs(qb) - 1;
                    // every lane walks its own quad; only lane Q's result is kept
                    AT ea = exclL + (lane == 0 ? AT(0) : qe);
                    AT Pj32 = AT(0), Pp32 = AT(0);
                    int E = -1;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const AT na = ea + xv[q];
                        const bool hit = (E < 0) && (xv[q] > AT(0)) && (na > t);
                        Pj32 = hit ? na : Pj32;
                        Pp32 = hit ? ea : Pp32;
                        E = hit ? q : E;
                        ea = na;
                    }
                    const double Pj = static_cast<double>(Pj32);
                    const double Pprev = static_cast<double>(Pp32);
                    const int Jc = cbaseL + 4 * lane + E;
                    const bool mine = (lane == Q) && (E >= 0);
                    J = mine ? Jc : -1;
                    cert = mine && (Pj * lo_f > A) && (Pprev + e_rel * Pj < B) && Jc < n;
                }
            }
            TICK(2);
            // speculative refill, issued by the certifying lane itself: every
            // read of buf in this step has returned (its value fed the ballots)
            if (cert && step + 1 < n) {
                mbar_expect_tx(bar, row_bytes);
                tma_row(buf, wbase + static_cast<size_t>(J) * p.PW, row_bytes, bar);
            }
            const unsigned cb = __ballot_sync(kFull, cert);
            ok = cb != 0u;
            if (ok) {
                next = __shfl_sync(kFull, J, __ffs(cb) - 1);
                prefetched = step + 1 < n;
            }
        }
        TICK(3);
        if (!ok) { // middle tier: fp64 sums over the fp32 row still in smem
            if constexpr (kGroupWalk) u = __shfl_sync(kFull, ubatch, (step - 1) & 31);
            const int j2 = certify_fp64<WT, NV, MAXR, NAT>(buf, tabu, n, p.R, u, lane);
            if (j2 >= 0) {
                ok = true;
                next = j2;
                ++fb2;
            }
        }
        if (!ok) {
            if (prefetched) { // never set when !ok, kept for safety
                mbar_wait(bar, phase);
                phase ^= 1u;
                prefetched = false;
            }
            next = exact_walk(p.w64 + static_cast<size_t>(cur) * p.P64, tabu, n,
                              p.tabu_words, u, lane, chunk_start,
                              reinterpret_cast<double*>(buf), row_bytes & ~255u, bar, phase);
            phase ^= static_cast<uint32_t>(exact_walk_pieces(n, row_bytes & ~255u) & 1);
            ++fb;
        }
        TICK(4);
        // Every read of the shared tabu in this step has been consumed by a
        // ballot/shuffle, so lane 0 updates it without a barrier; the
        // __syncwarp before the next step's mbarrier wait orders it before
        // any later read.
        if constexpr (STREAM) {
            if (lane == 0) tabu[next >> 5] |= 1u << (next & 31);
            if (lane == (step & 31)) held = next;
            if ((step & 31) == 31 || step == s1 - 1) { // the chunk (or the run) closes
                const int s = (step & ~31) + lane;
                if (s >= s0 && s <= step) {
                    tour[s] = held;
                    p.host_tours[static_cast<size_t>(kl) * (n + 1) + s] = held;
                }
            }
        } else if (lane == 0) {
            tabu[next >> 5] |= 1u << (next & 31);
            tour[step] = next;
        }
        cur = next;
        TICK(5);
    }
#if ACO_TIMING
    if (lane == 0 && p.timing)
        for (int i = 0; i < 7; ++i) atomicAdd(p.timing + i, ph[i]);
#endif
#undef TICK
    a.cur = cur;
    a.prefetched = prefetched;
}

// HI: high-occupancy launch (the issue-lean step: in-place scans, predicated
// sequential group sums)
template <typename WT, int NV, int MAXR, bool STREAM = false, bool HI = false, bool NAT = false>
__global__ void __launch_bounds__(32, MAXR == 1 ? 17 : 12) k_construct_roulette(ConstructParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    uint32_t* tabu = reinterpret_cast<uint32_t*>(smem_raw + 128 + static_cast<size_t>(p.PW) * sizeof(WT));
    const int lane = threadIdx.x & 31;
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    uint32_t phase = 0;
    unsigned long long fb = 0, fb2 = 0;
    for (int kl = blockIdx.x; kl < p.mloc; kl += gridDim.x) {
        RouletteAnt a;
        roulette_begin(p, a, kl, tabu, lane, STREAM);
        roulette_steps<WT, NV, MAXR, STREAM, HI, HI, NAT>(p, a, 1, p.n, smem_raw, phase, fb, fb2);
        roulette_end(p, a, lane, STREAM);
    }
    if (lane == 0) {
        if (fb) atomicAdd(p.fallbacks, fb);
        if (fb2) atomicAdd(p.tier2, fb2);
    }
}

// ---------------------------------------------------------------------------
// Relay variant of the fp32 single-round roulette.  With q = floor(m / SMs)
// warps on every SM and E = m - q*SMs leftover ants, the plain launch puts a
// (q+1)-th warp on E SMs; that warp shares an SM sub-partition (5 warps on
// one scheduler at q = 16) and holds the whole kernel back.  Here the grid is
// q*SMs warps, warp w builds ant w, and each leftover ant x is built in K
// segments by warps x, x+E, .., x+(K-1)E: warp x+iE runs its own ant up to
// the segment's first step, waits for segment i-1 to be handed over (building
// its own ant meanwhile), builds the segment, hands the tabu set and current
// city on, and finishes its own ant.  Every warp's work is the same steps of
// the same ants with the same draws, so tours are identical to the plain
// kernel's.  All runs of steps go through ONE inlined call site of the step
// loop (a small state machine picks the ant and the step range), so the hot
// loop compiles like the plain kernel's; only the run boundaries touch the
// two ants' state in local memory.
__device__ __forceinline__ void roulette_drain(RouletteAnt& a, uint64_t* bar, uint32_t& phase) {
    if (a.prefetched) { // a speculative row for this ant is in flight
        mbar_wait(bar, phase);
        phase ^= 1u;
        a.prefetched = false;
    }
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* q) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(q) : "memory");
    return v;
}

template <int NV, bool STREAM, bool HI = true>
__global__ void __launch_bounds__(32, 16) k_construct_roulette_relay(ConstructParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    uint32_t* tabu_own = reinterpret_cast<uint32_t*>(smem_raw + 128 + static_cast<size_t>(p.PW) * sizeof(float));
    // after chunk_start (single-round rows have no gsum area)
    uint32_t* tabu_rel = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(tabu_own + p.tabu_words) +
                                                     ((p.n + 31) >> 5));
    const int lane = threadIdx.x & 31;
    const int n = p.n;
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    uint32_t phase = 0;
    unsigned long long fb = 0, fb2 = 0;
    const int kl = blockIdx.x; // grid == relay_W: one own ant per warp
    const int rx = kl % p.relay_E, ri = kl / p.relay_E;
    const bool has_seg = ri < p.relay_K;
    const int seg_begin = has_seg ? relay_bound(ri, p.relay_K, n) : n;
    const int seg_end = has_seg ? relay_bound(ri + 1, p.relay_K, n) : n;
    const unsigned long long stamp = (p.relay_epoch << 20) | static_cast<unsigned>(ri);
    RouletteAnt ants[2]; // [0] own ant, [1] the relayed ant during the segment
    roulette_begin(p, ants[0], kl, tabu_own, lane, STREAM);
    int s = 1;                     // the own ant's next step
    int stage = has_seg ? 0 : 3;   // 0 own before the segment, 1 segment, 2 own after, 3 own only
    for (;;) {
        int which = 0, s0 = s, s1 = n;
        if (stage == 0) {
            if (s < seg_begin) {
                s1 = seg_begin;
            } else {
                bool ready = ri == 0;
                if (!ready) {
                    unsigned long long f = 0;
                    if (lane == 0) f = ld_acquire_u64(p.relay_flag + rx);
                    ready = __shfl_sync(kFull, f, 0) == stamp;
                }
                if (!ready) { // build the own ant one step further meanwhile
                    if (s >= n) {
                        __nanosleep(256);
                        continue;
                    }
                    s1 = s + 1;
                } else {
                    if (ri > 0) (void)ld_acquire_u64(p.relay_flag + rx); // order every lane's reads
                    roulette_drain(ants[0], bar, phase);
                    RouletteAnt& r = ants[1];
                    if (ri == 0) {
                        roulette_begin(p, r, p.relay_W + rx, tabu_rel, lane, STREAM);
                    } else {
                        r.kl = p.relay_W + rx;
                        r.kg = static_cast<uint32_t>(p.ant_begin + r.kl);
                        r.tour = p.tours + static_cast<size_t>(r.kl) * (n + 1);
                        r.tabu = tabu_rel;
                        r.prefetched = false;
                        const uint32_t* src = p.relay_tabu + static_cast<size_t>(rx) * p.tabu_words;
                        for (int wd = lane; wd < p.tabu_words; wd += 32) tabu_rel[wd] = __ldcg(src + wd);
                        r.cur = __ldcg(p.relay_cur + rx);
                        __syncwarp();
                    }
                    which = 1;
                    s0 = seg_begin;
                    s1 = seg_end;
                    stage = 1;
                }
            }
        } else if (stage == 1) { // segment built: hand it over (or close the tour)
            RouletteAnt& r = ants[1];
            roulette_drain(r, bar, phase);
            __syncwarp();
            if (seg_end == n) {
                roulette_end(p, r, lane, STREAM);
                if (ACO_FUSED_TAIL_BUILD && p.len_out) tour_tail(p, r.tour, r.kl, lane);
            } else {
                uint32_t* dst = p.relay_tabu + static_cast<size_t>(rx) * p.tabu_words;
                for (int wd = lane; wd < p.tabu_words; wd += 32) __stcg(dst + wd, tabu_rel[wd]);
                if (lane == 0) __stcg(p.relay_cur + rx, r.cur);
                __threadfence();
                __syncwarp();
                if (lane == 0)
                    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.relay_flag + rx),
                                 "l"(stamp + 1)
                                 : "memory");
            }
            stage = 2;
            if (s >= n) break;
        } else if (stage == 2) {
            break;
        } else {
            stage = 2;
        }
        roulette_steps<float, NV, 1, STREAM, true, HI>(p, ants[which], s0, s1, smem_raw, phase, fb, fb2);
        if (which == 0) s = s1;
    }
    roulette_end(p, ants[0], lane, STREAM);
    // fused tour tail (lengths, 1/C_k, succ/pred): the relay kernel has the
    // register room the plain one lacks (128 vs 96)
    if (ACO_FUSED_TAIL_BUILD && p.len_out) tour_tail(p, ants[0].tour, ants[0].kl, lane);
    if (lane == 0) {
        if (fb) atomicAdd(p.fallbacks, fb);
        if (fb2) atomicAdd(p.tier2, fb2);
    }
}

// ---------------------------------------------------------------------------
// Full-row roulette for rows too long for the streamed-row layouts (n beyond
// 8 rounds of 32 lanes x 80 cities) or on request (ACO_ROULETTE_EXACT=1):
// every step is the exact replay of select_next_roulette (exact_walk: the
// fp64 row staged through shared memory in TMA pieces, every lane folding
// every weight in ascending order).  Slower, but any n.
__global__ void __launch_bounds__(32) k_construct_roulette_exact(ConstructParams p, uint32_t stage_bytes) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    double* stage = reinterpret_cast<double*>(smem_raw + 128);
    uint32_t* tabu = reinterpret_cast<uint32_t*>(smem_raw + 128 + stage_bytes);
    double* chunk_start = reinterpret_cast<double*>(tabu + p.tabu_words);
    const int lane = threadIdx.x & 31;
    const int n = p.n;
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    uint32_t phase = 0;
    const uint32_t flip = static_cast<uint32_t>(exact_walk_pieces(n, stage_bytes) & 1);
    for (int kl = blockIdx.x; kl < p.mloc; kl += gridDim.x) {
        const uint32_t kg = static_cast<uint32_t>(p.ant_begin + kl);
        int32_t* tour = p.tours + static_cast<size_t>(kl) * (n + 1);
        tabu_init(tabu, p.tabu_words, n, lane);
        const int start = start_city(p, kg);
        __syncwarp();
        if (lane == 0) {
            tabu[start >> 5] |= 1u << (start & 31);
            tour[0] = start;
        }
        __syncwarp();
        int cur = start;
        double ubatch = 0.0;
        for (int step = 1; step < n; ++step) {
            if (((step - 1) & 31) == 0)
                ubatch = philox_uniform(p.seed, p.iteration, kg, static_cast<uint32_t>(step + lane), 0);
            const double u = __shfl_sync(kFull, ubatch, (step - 1) & 31);
            const int next = exact_walk(p.w64 + static_cast<size_t>(cur) * p.P64, tabu, n,
                                        p.tabu_words, u, lane, chunk_start, stage, stage_bytes, bar,
                                        phase);
            phase ^= flip;
            __syncwarp();
            if (lane == 0) {
                tabu[next >> 5] |= 1u << (next & 31);
                tour[step] = next;
            }
            __syncwarp();
            cur = next;
        }
        if (lane == 0) tour[n] = start;
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// NN-list roulette (select_next_nn, construction.hpp:73-121).  Lane q holds
// list member q (nn <= 32 per pass) and its fp64 weight (0 if visited).  One
// fold over the list: every lane adds the broadcast weights in LIST order —
// the reference's own sequential sums — and lane q keeps the prefix after
// member q, so total = last prefix, and the walk's first crossing is one
// ballot (a visited member adds +0.0 and can never be the first crossing).
// No certification is needed.  When the whole list is visited, the fallback
// is the exact (value, lowest index) argmax over all unvisited cities
// (construction.hpp:108-120), which consumes no draw; it streams the fp64
// row with 8 independent 16-byte loads per lane in flight.
#ifndef ACO_NN_MINB
#define ACO_NN_MINB 32 // resident warps per SM the register budget must allow (64 registers, no spills)
#endif
#ifndef ACO_NN_SPEC_MINB
#define ACO_NN_SPEC_MINB 28 // the same for the latency-bound (SPEC) launches (<= 12 ants per SM)
#endif
// SPEC: the crossing candidate's list is requested before its certification
// (for latency-bound launches; that variant is held to 64 registers)
// FAST32: nn <= 32 with the row-scaled fp32 list weights (the fast path)
template <bool SPEC, bool FAST32 = true>
__global__ void __launch_bounds__(32, SPEC ? ACO_NN_SPEC_MINB : ACO_NN_MINB) k_construct_nn(ConstructParams p) {
    extern __shared__ uint32_t smem_tabu[];
    uint32_t* tabu = smem_tabu;

    const int lane = threadIdx.x & 31;
    const int n = p.n, nn = p.nn;
    // fp32 fast-path certification constants (outward-rounded, formed on the
    // host: nn_certify_constants) come straight from the parameter bank, so
    // the hot loop holds no registers for them
    const float nn_e32 = p.nn_e32, nn_lo32 = p.nn_lo32, nn_ce = p.nn_ce, nn_absq = p.nn_absq;
    for (int kl = blockIdx.x; kl < p.mloc; kl += gridDim.x) {
        const uint32_t kg = static_cast<uint32_t>(p.ant_begin + kl);
        int32_t* tour = p.tours + static_cast<size_t>(kl) * (n + 1);
        tabu_init(tabu, p.tabu_words, n, lane);
        const int start = start_city(p, kg);
        __syncwarp();
        if (lane == 0) {
            tabu[start >> 5] |= 1u << (start & 31);
            tour[0] = start;
        }
        __syncwarp();
        int cur = start;
        unsigned long long fb = 0, fb_full = 0;
        double ubatch = 0.0;
        float ub_up = 0.f, ub_dn = 0.f;
        // fp32 fast path: the current city's list (ids, scaled weights) is
        // loaded as soon as that city is chosen, one step ahead, so the L2
        // round trip overlaps the previous step's bookkeeping
        constexpr bool fast32 = FAST32;
        int jpre = -1;
        float wpre = 0.f;
        // SPEC: the crossing candidate's list is requested before its
        // certification
        int jg = -1;
        int jspec = -1;
        float wspec = 0.f;
        // kHold (full-occupancy launches): the open 32-entry chunk of the
        // tour (and of the list positions) is held in the lanes — lane
        // (s & 31) holds tour[s] / qpos[s-1] — and stored coalesced when the
        // chunk closes, instead of lane 0 storing every step
        constexpr bool kHold = !SPEC;
        int held_t = 0, held_q = 0;
        if (fast32 && lane < nn) {
            {
                const int2 rec = p.choice_nn32[static_cast<unsigned>(start * nn + lane)];
                jpre = rec.x;
                wpre = __int_as_float(rec.y);
            }
        }
        for (int step = 1; step < n; ++step) {
            const double* __restrict__ row = p.w64 + static_cast<size_t>(cur) * p.P64;
            const int32_t* nb = p.nn_lists + static_cast<size_t>(cur) * nn;
            const double* wn = p.choice_nn + static_cast<size_t>(cur) * nn;
            // Draw 0 of steps step..step+31: lane i holds step + i
            // (rng.hpp:74-80), kept in fp64 and as the float pair that
            // brackets it (rounded down / up): the fast path broadcasts the
            // pair (two 32-bit shuffles, no conversions per step), the exact
            // paths the fp64 draw
            if (((step - 1) & 31) == 0) {
                ubatch = philox_uniform(p.seed, p.iteration, kg,
                                        static_cast<uint32_t>(step + lane), 0);
                ub_up = __double2float_ru(ubatch);
                ub_dn = __double2float_rd(ubatch);
            }
            const float u_up = __shfl_sync(kFull, ub_up, (step - 1) & 31);
            const float u_dn = __shfl_sync(kFull, ub_dn, (step - 1) & 31);
            int next = -1;
            int qsel = 255;         // list position of next (255: not from the list)
            bool exhausted = false; // every list member visited: argmax fallback
            if (fast32) {
                // Fast path on the row-scaled fp32 copy of the list weights
                // (k_rows: the list maximum scaled into [2^112, 2^113) by an
                // exact power of two, so scaled and unscaled comparisons
                // agree): one fp32 warp scan, then the crossing J is
                // CERTIFIED against the reference's fp64 sequential sums —
                // |P_q - X_q| <= e*X_q + nn*2^-150 with e covering the fp32
                // quantisation (1 ulp), the 5 scan levels and the
                // reference's own nn sequential fp64 adds; thresholds are
                // rounded outward so the fp32 compares imply the exact ones.
                // T == 0 (possible through fp32 underflow) and uncertain
                // steps take the exact fp64 fold below.
                const int q = lane;
                int j = -1;
                float w = 0.f;
                bool un = false;
                if (q < nn) {
                    j = jpre;
                    un = !tabu_test(tabu, j);
                    w = un ? wpre : 0.f;
                }
                const unsigned unb = __ballot_sync(kFull, un);
                if (!unb) {
                    exhausted = true;
                } else {
                    const float P = warp_inclusive_scan<!SPEC>(w);
                    const float T = __shfl_sync(kFull, P, 31);
                    const float Eu = __shfl_up_sync(kFull, P, 1); // every lane shuffles
                    const float E = lane == 0 ? 0.f : Eu;
                    // the candidate threshold only (the certification
                    // below brackets u between u_dn and u_up)
                    const float t32 = __fmul_rn(u_dn, T);
                    const unsigned cr = __ballot_sync(kFull, q < nn && w > 0.f && P > t32 && T > 0.f);
                    if (cr) {
                        const int J = __ffs(cr) - 1;
                        const float PJ = __shfl_sync(kFull, P, J);
                        const float EJ = __shfl_sync(kFull, E, J);
                        const int Jc = __shfl_sync(kFull, j, J);
                        if (SPEC && lane < nn && step + 1 < n) {
                            // the candidate's list, requested before its
                            // certification (which almost always passes)
                            jg = Jc;
                            {
                                const int2 rec = p.choice_nn32[static_cast<unsigned>(Jc * nn + lane)];
                                jspec = rec.x;
                                wspec = __int_as_float(rec.y);
                            }
                        }
                        // thresholds in fp32, every operation rounded
                        // outward: A32 >= u*T + Mt + 2*abs, B32 <= u*T - Mt -
                        // 2*abs, Mt >= (e + 4*2^-24) * u * (T(1+2^-16) + abs)
                        // + abs (|t_ref - u*T| <= Mt)
                        const float Thi = __fadd_ru(__fmul_ru(T, 1.0f + 0x1.0p-16f), nn_absq);
                        const float Mt = __fadd_ru(__fmul_ru(nn_ce, __fmul_ru(u_up, Thi)), nn_absq);
                        const float A32 = __fadd_ru(__fadd_ru(__fmul_ru(u_up, T), Mt), 2.0f * nn_absq);
                        const float B32 = __fsub_rd(__fsub_rd(__fmul_rd(u_dn, T), Mt), 2.0f * nn_absq);
                        if (__fmul_rd(PJ, nn_lo32) > A32 && __fadd_ru(EJ, __fmul_ru(nn_e32, PJ)) < B32) {
                            next = Jc;
                            qsel = J;
                        }
                    }
                }
            } else if (nn <= 32) {
                const double u = __shfl_sync(kFull, ubatch, (step - 1) & 31);
                // Fast path: one fp64 warp scan instead of the sequential
                // fold, then CERTIFY the crossing against the reference's
                // sequential sums (as in k_construct_roulette): every scan
                // prefix P_q and the reference's S_q are within e*X_q of the
                // exact prefix X_q (e: 5 scan levels + nn sequential adds,
                // all summands >= 0), and t_ref = fl(u*S_n) within Mt of
                // t = u*T.  Uncertain steps (~never at e ~ 2^-47) take the
                // exact fold below.
                const int q = lane;
                int j = -1;
                double w = 0.0;
                bool un = false;
                if (q < nn) {
                    j = nb[q];
                    const double wq0 = wn[q];
                    un = !tabu_test(tabu, j);
                    w = un ? wq0 : 0.0;
                }
                const unsigned unb = __ballot_sync(kFull, un);
                if (!unb) {
                    exhausted = true;
                } else {
                    double P = w;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const double y = __shfl_up_sync(kFull, P, off);
                        if (lane >= off) P += y;
                    }
                    const double T = __shfl_sync(kFull, P, 31);
                    if (!(T > 0.0)) {
                        qsel = __ffs(unb) - 1;
                        next = __shfl_sync(kFull, j, qsel); // :89-92, exact
                    } else {
                        const double Eu = __shfl_up_sync(kFull, P, 1); // every lane shuffles
                        const double E = lane == 0 ? 0.0 : Eu;
                        const double t = u * T;
                        const unsigned cr = __ballot_sync(kFull, q < nn && w > 0.0 && P > t);
                        if (cr) {
                            const int J = __ffs(cr) - 1;
                            const double PJ = __shfl_sync(kFull, P, J);
                            const double EJ = __shfl_sync(kFull, E, J);
                            const double e = 48.0 * 0x1.0p-53;
                            const double Mt = (e + 0x1.0p-51) * u * T * (1.0 + 0x1.0p-16) + 0x1.0p-1074;
                            const int jJ = __shfl_sync(kFull, j, J);
                            if (PJ * (1.0 - e) > t + Mt && EJ + e * T < t - Mt) {
                                next = jJ;
                                qsel = J;
                            }
                        }
                    }
                }
            }
            // exact sequential fold (only when the fast path left the step
            // open): lane q of pass k holds member 32k+q
            if (next < 0 && !exhausted) {
            const double u = __shfl_sync(kFull, ubatch, (step - 1) & 31);
            double acc = 0.0;
            int first_un = -1, last_pos = -1, first_un_q = 255, last_pos_q = 255;
            double mine[2] = {0.0, 0.0};
            int jm[2] = {-1, -1};
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int q0 = 32 * k;
                if (q0 < nn) {
                    const int q = q0 + lane;
                    int j = -1;
                    double w = 0.0;
                    bool un = false;
                    if (q < nn) {
                        // id and weight issued together: one L2 round trip per step
                        j = nb[q];
                        const double wq0 = wn[q];
                        un = !tabu_test(tabu, j);
                        w = un ? wq0 : 0.0;
                    }
                    jm[k] = j;
                    const unsigned unb = __ballot_sync(kFull, un);
                    const unsigned pob = __ballot_sync(kFull, un && w > 0.0);
                    if (first_un < 0 && unb) {
                        first_un_q = q0 + __ffs(unb) - 1;
                        first_un = __shfl_sync(kFull, j, __ffs(unb) - 1);
                    }
                    if (pob) {
                        last_pos_q = q0 + 31 - __clz(pob);
                        last_pos = __shfl_sync(kFull, j, 31 - __clz(pob));
                    }
                    // lanes >= nn carry w = +0.0, so folding all 32 is exact
                    double wq[32];
#pragma unroll
                    for (int s2 = 0; s2 < 32; ++s2) wq[s2] = __shfl_sync(kFull, w, s2);
#pragma unroll
                    for (int s2 = 0; s2 < 32; ++s2) {
                        acc += wq[s2];
                        mine[k] = (s2 == lane) ? acc : mine[k];
                    }
                }
            }
            if (first_un >= 0) {
                const double total = acc;
                if (!(total > 0.0)) {
                    next = first_un;                                     // :89-92
                    qsel = first_un_q;
                } else {
                    const double target = u * total;                     // :93
#pragma unroll
                    for (int k = 0; k < 2 && next < 0; ++k) {
                        if (32 * k < nn) {
                            const unsigned cr = __ballot_sync(kFull, lane + 32 * k < nn && mine[k] > target);
                            if (cr) {
                                next = __shfl_sync(kFull, jm[k], __ffs(cr) - 1);
                                qsel = 32 * k + __ffs(cr) - 1;
                            }
                        }
                    }
                    if (next < 0) { // :103-105
                        next = last_pos >= 0 ? last_pos : first_un;
                        qsel = last_pos >= 0 ? last_pos_q : first_un_q;
                    }
                }
            }
            }
            if (next < 0) {
                // argmax over all unvisited, lowest index on ties (:108-120):
                // first the row's top-K cache (k_row_topk): its first
                // unvisited entry IS the argmax; a full scan only when every
                // cached entry is visited (or the row's cache is invalid).
                ++fb;
                if (p.topk) {
                    const int32_t* tk = p.topk + static_cast<size_t>(cur) * p.topk_k;
                    // 128 entries (4 loads per lane in flight) at a time
                    for (int r0 = 0; r0 < p.topk_k && next < 0; r0 += 128) {
                        int ids[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            ids[r] = r0 + 32 * r < p.topk_k ? tk[r0 + 32 * r + lane] : -1;
                        if (r0 == 0 && __shfl_sync(kFull, ids[0], 0) == -2) break; // invalid row: scan
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const bool un = ids[r] >= 0 && !tabu_test(tabu, ids[r]);
                            const unsigned b = __ballot_sync(kFull, un);
                            if (b && next < 0) next = __shfl_sync(kFull, ids[r], __ffs(b) - 1);
                        }
                        if (__shfl_sync(kFull, ids[3], 31) < 0) break; // end of the list (n < K)
                    }
                    if (next >= 0) qsel = 255; // not from the list
                }
                if (next < 0) {
                ++fb_full;
                double bw = -1.0;
                int bj = -1;
                const double2* r2 = reinterpret_cast<const double2*>(row);
                const int n2 = (n + 1) >> 1;
                if (4 * (n - step) < n) {
                    // few cities left: gather only the unvisited ones (8 in flight)
                    for (int w0 = 0; w0 < p.tabu_words; w0 += 32) {
                        const int wd = w0 + lane;
                        uint32_t freeb = wd < p.tabu_words ? ~tabu[wd] : 0u;
                        while (freeb) {
                            int js[8];
                            double vs[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                js[i] = -1;
                                if (freeb) {
                                    js[i] = wd * 32 + __ffs(freeb) - 1;
                                    freeb &= freeb - 1;
                                }
                            }
#pragma unroll
                            for (int i = 0; i < 8; ++i) vs[i] = js[i] >= 0 ? __ldg(row + js[i]) : -1.0;
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                if (js[i] >= 0 && vs[i] > bw) { bw = vs[i]; bj = js[i]; }
                        }
                    }
                } else
                for (int b0 = 0; b0 < n2; b0 += 32 * 8) {
                    double2 v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int k2 = b0 + i * 32 + lane;
                        v[i] = k2 < n2 ? __ldg(r2 + k2) : make_double2(-1.0, -1.0);
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int j0 = 2 * (b0 + i * 32 + lane);
                        if (j0 < n && !tabu_test(tabu, j0) && v[i].x > bw) { bw = v[i].x; bj = j0; }
                        if (j0 + 1 < n && !tabu_test(tabu, j0 + 1) && v[i].y > bw) { bw = v[i].y; bj = j0 + 1; }
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ow = __shfl_xor_sync(kFull, bw, off);
                    const int oj = __shfl_xor_sync(kFull, bj, off);
                    if (oj >= 0 && (bj < 0 || ow > bw || (ow == bw && oj < bj))) { bw = ow; bj = oj; }
                }
                next = bj;
                }
            }
            if (fast32 && step + 1 < n) {
                if (SPEC && next == jg) { // the speculated list is the one
                    jpre = jspec;
                    wpre = wspec;
                } else if (lane < nn) {
                    {
                        const int2 rec = p.choice_nn32[static_cast<unsigned>(next * nn + lane)];
                        jpre = rec.x;
                        wpre = __int_as_float(rec.y);
                    }
                }
            }
            jg = -1;
            if constexpr (kHold) {
                if (lane == 0) tabu[next >> 5] |= 1u << (next & 31);
                if (lane == (step & 31)) {
                    held_t = next;
                    held_q = qsel;
                }
                if ((step & 31) == 31 || step == n - 1) {
                    const int s = (step & ~31) + lane;
                    if (s >= 1 && s <= step) {
                        tour[s] = held_t;
                        if (p.qpos) p.qpos[static_cast<size_t>(kl) * n + s - 1] = static_cast<uint8_t>(held_q);
                    }
                }
            } else if (lane == 0) {
                tabu[next >> 5] |= 1u << (next & 31);
                tour[step] = next;
                if (p.qpos) p.qpos[static_cast<size_t>(kl) * n + step - 1] = static_cast<uint8_t>(qsel);
            }
            __syncwarp();
            cur = next;
        }
        if (lane == 0) {
            tour[n] = start;
            if (p.qpos) p.qpos[static_cast<size_t>(kl) * n + n - 1] = 255; // the closing edge
            if (fb) atomicAdd(p.argmax_fallbacks, fb);
            if (fb_full) atomicAdd(p.fallbacks, fb_full);
        }
        __syncwarp();
        if (ACO_FUSED_TAIL_BUILD && p.len_out) tour_tail(p, tour, kl, lane);
    }
}

// ---------------------------------------------------------------------------
// Data-parallel "independent roulette" (select_next_data_parallel,
// construction.hpp:129-162; the paper's Fig. 1): city j scores w_j * u_j with
// its own draw (draw index j), the winner is the lowest-index maximum over
// the unvisited cities (tile reduction order does not change it), and a
// non-positive best falls back to the lowest unvisited city.
__global__ void __launch_bounds__(128) k_construct_data_parallel(ConstructParams p) {
    extern __shared__ uint32_t smem_tabu[]; // [4][tabu_words] tabu, then [4][1024] lists
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* tabu = smem_tabu + wib * p.tabu_words;
    int* list = reinterpret_cast<int*>(smem_tabu + 4 * p.tabu_words) + wib * 1024;
    const int n = p.n;
    for (int kl = blockIdx.x * 4 + wib; kl < p.mloc; kl += gridDim.x * 4) {
        const uint32_t kg = static_cast<uint32_t>(p.ant_begin + kl);
        int32_t* tour = p.tours + static_cast<size_t>(kl) * (n + 1);
        tabu_init(tabu, p.tabu_words, n, lane);
        const int start = start_city(p, kg);
        __syncwarp();
        if (lane == 0) {
            tabu[start >> 5] |= 1u << (start & 31);
            tour[0] = start;
        }
        __syncwarp();
        int cur = start;
        for (int step = 1; step < n; ++step) {
            const double* __restrict__ row = p.w64 + static_cast<size_t>(cur) * p.P64;
            double bs = 0.0;
            int bj = -1;
            // Only unvisited cities draw and score: 1024 cities (32 tabu
            // words) at a time, their unvisited indices are compacted in
            // ascending order into the warp's list (popc + warp scan), then
            // the lanes take list entries round-robin — every lane still
            // meets its cities in ascending order, so "first max per lane,
            // then lowest index among equal maxima" is unchanged.
            for (int w0 = 0; w0 < p.tabu_words; w0 += 32) {
                const int wd = w0 + lane;
                uint32_t ub = wd < p.tabu_words ? ~tabu[wd] : 0u;
                const int cnt = __popc(ub);
                int incl = cnt;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int y = __shfl_up_sync(kFull, incl, off);
                    if (lane >= off) incl += y;
                }
                const int total = __shfl_sync(kFull, incl, 31);
                int pos = incl - cnt;
                while (ub) {
                    list[pos++] = wd * 32 + __ffs(ub) - 1;
                    ub &= ub - 1;
                }
                __syncwarp();
                for (int r = lane; r < total; r += 32) {
                    const int j = list[r];
                    const double u = philox_uniform(p.seed, p.iteration, kg,
                                                    static_cast<uint32_t>(step), static_cast<uint32_t>(j));
                    const double s = row[j] * u;
                    if (bj < 0 || s > bs) { bs = s; bj = j; }
                }
                __syncwarp();
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double os = __shfl_xor_sync(kFull, bs, off);
                const int oj = __shfl_xor_sync(kFull, bj, off);
                if (oj >= 0 && (bj < 0 || os > bs || (os == bs && oj < bj))) { bs = os; bj = oj; }
            }
            int next = bj;
            if (!(bs > 0.0)) next = lowest_unvisited(tabu, p.tabu_words, lane);
            if (lane == 0) {
                tabu[next >> 5] |= 1u << (next & 31);
                tour[step] = next;
            }
            __syncwarp();
            cur = next;
        }
        if (lane == 0) tour[n] = start;
        __syncwarp();
    }
}

} // namespace acob200
