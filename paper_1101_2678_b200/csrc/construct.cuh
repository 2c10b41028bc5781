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

__host__ __device__ __forceinline__ int stream_pos(int c, int C, int V) {
    const int R32 = 32 * C;
    const int r = c / R32, rem = c - r * R32;
    const int l = rem / C, e = rem - l * C;
    const int t = e / V, q = e - t * V;
    return r * R32 + (t * 32 + l) * V + q;
}

__host__ __device__ __forceinline__ int stream_city(int p, int C, int V) {
    const int R32 = 32 * C;
    const int r = p / R32, rem = p - r * R32;
    const int t = rem / (32 * V), rem2 = rem - t * 32 * V;
    const int l = rem2 / V, q = rem2 - l * V;
    return r * R32 + l * C + t * V + q;
}

struct ConstructParams {
    const void* w;           // streamed weights (float or double), row pitch PW
    const double* w64;       // natural fp64 choice, row pitch P64 (exact walk, nn)
    const int32_t* nn_lists; // n x nn (nn selection)
    int32_t* tours;          // mloc x (n+1)
    unsigned long long* fallbacks;
    unsigned long long* argmax_fallbacks;
    int n, P64, PW, R, nn;
    int ant_begin, mloc;
    int random_start;
    int theta;
    int tabu_words; // per warp; >= PW/32 + 2
    uint32_t iteration;
    uint64_t seed;
};

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
// reference's `continue`.
__device__ __noinline__ int exact_walk(const double* __restrict__ row, const uint32_t* tabu,
                                       int n, int words, double u, int lane) {
    double acc = 0.0;
    double w_next = 0.0;
    {
        const int j = lane;
        if (j < n && !tabu_test(tabu, j)) w_next = row[j];
    }
    for (int base = 0; base < n; base += 32) {
        const double w = w_next;
        const int j = base + 32 + lane;
        w_next = (j < n && !tabu_test(tabu, j)) ? row[j] : 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) acc += __shfl_sync(kFull, w, q);
    }
    if (!(acc > 0.0)) return lowest_unvisited(tabu, words, lane); // total <= 0 (:52)
    const double target = u * acc;                                  // :54
    double a2 = 0.0;
    int last_positive = -1;
    for (int base = 0; base < n; base += 32) {
        const int j = base + lane;
        const double w = (j < n && !tabu_test(tabu, j)) ? row[j] : 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const double x = __shfl_sync(kFull, w, q);
            if (x > 0.0) last_positive = base + q;
            a2 += x;
            if (a2 > target) return base + q; // warp-uniform
        }
    }
    if (last_positive >= 0) return last_positive; // :66
    return lowest_unvisited(tabu, words, lane);
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

// ---------------------------------------------------------------------------
// Roulette over the full row, one warp (= one CTA) per ant.  Per step:
//   lane 0 issues one cp.async.bulk of the row (PW * sizeof(WT) bytes) into
//   shared memory; all lanes draw u (Philox) while it flies; after the
//   mbarrier completes, lane l reads its contiguous chunk (C cities, NV
//   conflict-free 128-bit LDS), masks it with its tabu window, tree-sums it in
//   groups of 4 vectors, and the warp scans the lane sums in fp64.  The chunk
//   holding the crossing is then re-scanned COOPERATIVELY (EPL elements per
//   lane, warp scan, ballot) to locate j*, which is certified or replayed.
// NV = 128-bit vectors per lane per round, C = NV*V, MAXR = max rounds.
template <typename WT, int NV, int MAXR>
__global__ void __launch_bounds__(32, MAXR == 1 ? 20 : 12) k_construct_roulette(ConstructParams p) {
    using VT = typename VecOf<WT>::T;
    constexpr int V = VecOf<WT>::V;
    constexpr int C = NV * V;
    constexpr int NWIN = (C + 31) / 32;
    constexpr int GV = 4;                              // vectors per tree group
    constexpr int NG = (NV + GV - 1) / GV;             // groups per chunk
    constexpr int D1 = ceil_log2<GV * V>() + ceil_log2<NG>();
    constexpr int GE = GV * V;                         // cities per group
    constexpr bool F32 = sizeof(WT) == 4;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    WT* buf = reinterpret_cast<WT*>(smem_raw + 128);
    uint32_t* tabu = reinterpret_cast<uint32_t*>(smem_raw + 128 + static_cast<size_t>(p.PW) * sizeof(WT));
    WT* gsum = reinterpret_cast<WT*>(tabu + p.tabu_words); // [MAXR][NG][32] lane group sums
    const int lane = threadIdx.x & 31;
    const int n = p.n;
    const WT* __restrict__ wbase = static_cast<const WT*>(p.w);
    const uint32_t row_bytes = static_cast<uint32_t>(p.PW * sizeof(WT));

    // Certification constants (header comment); bounds relative to Thi.
    // e: relative error of every prefix estimate P_j (ours) plus the
    // reference's own sequential-sum error gamma_n, both relative to the
    // exact prefix X_j; abs_q: fp32 underflow (2^-150 per element, doubled).
    const double e_rel = ((F32 ? (1.0 + D1) * 0x1.0p-24 : D1 * 0x1.0p-53) +
                          (double)(8 + MAXR + NG + 8 + 8) * 0x1.0p-53 +
                          (double)(n + 2) * 0x1.0p-53) * (1.0 + 0x1.0p-20);
    const double abs_q = F32 ? (double)n * 0x1.0p-149 : 0.0;

    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    uint32_t phase = 0;

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
        int cur = start;
        unsigned long long fb = 0;

        for (int step = 1; step < n; ++step) {
            if (lane == 0) {
                fence_proxy_async_smem(); // generic reads of buf happen-before the refill
                mbar_expect_tx(bar, row_bytes);
                tma_row(buf, wbase + static_cast<size_t>(cur) * p.PW, row_bytes, bar);
            }
            const double u = philox_uniform(p.seed, p.iteration, kg, static_cast<uint32_t>(step), 0);
            __syncwarp();
            mbar_wait(bar, phase);
            phase ^= 1u;

            double incl[MAXR];
            double rtot[MAXR];
            double T = 0.0;
#pragma unroll
            for (int r = 0; r < MAXR; ++r) {
                incl[r] = 0.0;
                rtot[r] = 0.0;
                if (r < p.R) {
                    const int cbase = r * 32 * C + lane * C;
                    const int w0 = cbase >> 5, sh = cbase & 31;
                    uint32_t win[NWIN];
#pragma unroll
                    for (int i = 0; i < NWIN; ++i)
                        win[i] = __funnelshift_r(tabu[w0 + i], tabu[w0 + i + 1], sh);
                    const VT* rv = reinterpret_cast<const VT*>(buf + r * 32 * C) + lane;
                    WT gs[NG];
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        WT x[GV * V];
#pragma unroll
                        for (int tt = 0; tt < GV; ++tt) {
                            const int t = g * GV + tt;
                            if (t < NV) {
                                const VT v = rv[t * 32];
                                if constexpr (F32) {
                                    x[tt * 4 + 0] = v.x; x[tt * 4 + 1] = v.y;
                                    x[tt * 4 + 2] = v.z; x[tt * 4 + 3] = v.w;
                                } else {
                                    x[tt * 2 + 0] = v.x; x[tt * 2 + 1] = v.y;
                                }
                            } else {
#pragma unroll
                                for (int q = 0; q < V; ++q) x[tt * V + q] = WT(0);
                            }
                        }
#pragma unroll
                        for (int e = 0; e < GV * V; ++e) {
                            const int ee = g * GV * V + e;
                            if (ee < C && ((win[ee >> 5] >> (ee & 31)) & 1u)) x[e] = WT(0);
                        }
                        gs[g] = tree_sum<WT, GV * V>(x);
                        gsum[(r * NG + g) * 32 + lane] = gs[g];
                    }
                    double d = static_cast<double>(tree_sum<WT, NG>(gs));
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const double y = __shfl_up_sync(kFull, d, off);
                        if (lane >= off) d += y;
                    }
                    incl[r] = d;
                    rtot[r] = __shfl_sync(kFull, d, 31);
                    T += rtot[r];
                }
            }
            const double t = u * T;
            bool ok = (T > 0.0) && (T < 1e300);
            int next = -1;
            if (ok) {
                double base = 0.0, my = 0.0;
                int rs = -1;
#pragma unroll
                for (int r = 0; r < MAXR; ++r) {
                    if (r < p.R && rs < 0) {
                        if (base + rtot[r] > t) {
                            rs = r;
                            my = incl[r];
                        } else {
                            base += rtot[r];
                        }
                    }
                }
                const double prev_lane = __shfl_up_sync(kFull, my, 1);
                const unsigned bal = __ballot_sync(kFull, rs >= 0 && base + my > t);
                if (bal == 0u) {
                    ok = false;
                } else {
                    const int L = __ffs(bal) - 1;
                    const double start_acc = base + __shfl_sync(kFull, L == 0 ? 0.0 : prev_lane, L);
                    // 1) group of lane L's chunk holding the crossing: prefix of
                    //    its NG group sums (broadcast smem reads, fp64)
                    double gacc = start_acc, gbefore = start_acc;
                    int G = -1;
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        const double gv = static_cast<double>(gsum[(rs * NG + g) * 32 + L]);
                        const double na = gacc + gv;
                        if (G < 0 && na > t) {
                            G = g;
                            gbefore = gacc;
                        }
                        gacc = na;
                    }
                    int jstar = -1;
                    double Pj = 0.0, Pprev = 0.0;
                    if (G >= 0) {
                        // 2) the GE cities of that group: one per lane, fp64 scan
                        const int e = G * GE + lane;
                        const int cbase = rs * 32 * C + L * C;
                        double v = 0.0;
                        if (lane < GE && e < C && !tabu_test(tabu, cbase + e))
                            v = static_cast<double>(
                                buf[rs * 32 * C + ((e / V) * 32 + L) * V + (e % V)]);
                        double pin = v;
#pragma unroll
                        for (int off = 1; off < GE; off <<= 1) {
                            const double y = __shfl_up_sync(kFull, pin, off);
                            if (lane >= off) pin += y;
                        }
                        const double pup = __shfl_up_sync(kFull, pin, 1);
                        const unsigned b2 =
                            __ballot_sync(kFull, lane < GE && v > 0.0 && gbefore + pin > t);
                        if (b2) {
                            const int Lw = __ffs(b2) - 1;
                            jstar = cbase + G * GE + Lw;
                            Pj = gbefore + __shfl_sync(kFull, pin, Lw);
                            Pprev = gbefore + (Lw == 0 ? 0.0 : __shfl_sync(kFull, pup, Lw));
                        }
                    }
                    if (jstar < 0 || jstar >= n) {
                        ok = false;
                    } else {
                        // Certification (header comment), margins relative to t:
                        // |t_ref - t| <= Mt, s_j* >= Pj(1-e) - 2abs, s_prev <= Pprev(1+e) + 2abs.
                        const double Thi = T * (1.0 + 0x1.0p-20) + abs_q;
                        const double Mt = (e_rel + 0x1.0p-50) * (u * Thi) + abs_q;
                        ok = (Pj - e_rel * Pj - 2.0 * abs_q > t + Mt) &&
                             (Pprev + e_rel * Pprev + 2.0 * abs_q < t - Mt);
                        next = jstar;
                    }
                }
            }
            if (!ok) {
                next = exact_walk(p.w64 + static_cast<size_t>(cur) * p.P64, tabu, n,
                                  p.tabu_words, u, lane);
                ++fb;
            }
            __syncwarp();
            if (lane == 0) {
                tabu[next >> 5] |= 1u << (next & 31);
                tour[step] = next;
            }
            __syncwarp();
            cur = next;
        }
        if (lane == 0) {
            tour[n] = start;
            if (fb) atomicAdd(p.fallbacks, fb);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// NN-list roulette (select_next_nn, construction.hpp:73-121).  The <= nn
// candidate weights are gathered once (lane q holds list member q) and every
// lane folds them in LIST order, so the sums are the reference's own: no
// certification is needed.  When the whole list is visited, the fallback is
// the exact (value, lowest index) argmax over all unvisited cities
// (construction.hpp:108-120), which consumes no draw.
__global__ void __launch_bounds__(32, 16) k_construct_nn(ConstructParams p) {
    extern __shared__ uint32_t smem_tabu[];
    uint32_t* tabu = smem_tabu;
    const int lane = threadIdx.x & 31;
    const int n = p.n, nn = p.nn;
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
        unsigned long long fb = 0;
        for (int step = 1; step < n; ++step) {
            const double* __restrict__ row = p.w64 + static_cast<size_t>(cur) * p.P64;
            const int32_t* nb = p.nn_lists + static_cast<size_t>(cur) * nn;
            int next = -1;
            bool any = false;
            // candidates in chunks of 32 list members (nn is usually <= 32)
            double total = 0.0;
            for (int q0 = 0; q0 < nn; q0 += 32) {
                const int q = q0 + lane;
                int j = -1;
                double w = 0.0;
                bool un = false;
                if (q < nn) {
                    j = nb[q];
                    un = !tabu_test(tabu, j);
                    if (un) w = row[j];
                }
                any |= (__ballot_sync(kFull, un) != 0u);
                const int cnt = min(32, nn - q0);
                for (int s = 0; s < cnt; ++s) total += __shfl_sync(kFull, w, s);
            }
            if (any) {
                const double u = philox_uniform(p.seed, p.iteration, kg, static_cast<uint32_t>(step), 0);
                int first_un = -1, last_positive = -1;
                const double target = u * total;
                double acc = 0.0;
                for (int q0 = 0; q0 < nn && next < 0; q0 += 32) {
                    const int q = q0 + lane;
                    int j = -1;
                    double w = 0.0;
                    bool un = false;
                    if (q < nn) {
                        j = nb[q];
                        un = !tabu_test(tabu, j);
                        if (un) w = row[j];
                    }
                    const unsigned unb = __ballot_sync(kFull, un);
                    if (first_un < 0 && unb) first_un = __shfl_sync(kFull, j, __ffs(unb) - 1);
                    const int cnt = min(32, nn - q0);
                    for (int s = 0; s < cnt; ++s) {
                        const double x = __shfl_sync(kFull, w, s);
                        const int js = __shfl_sync(kFull, j, s);
                        if (next < 0 && ((unb >> s) & 1u)) {
                            if (x > 0.0) last_positive = js;
                            acc += x;
                            if (total > 0.0 && acc > target) next = js;
                        }
                    }
                }
                if (!(total > 0.0)) next = first_un;                 // :89-92
                else if (next < 0) next = last_positive >= 0 ? last_positive : first_un; // :103-105
            } else {
                // argmax over all unvisited, lowest index on ties (:108-120)
                double bw = -1.0;
                int bj = -1;
                for (int j = lane; j < n; j += 32) {
                    if (!tabu_test(tabu, j)) {
                        const double w = row[j];
                        if (w > bw) { bw = w; bj = j; }
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ow = __shfl_xor_sync(kFull, bw, off);
                    const int oj = __shfl_xor_sync(kFull, bj, off);
                    if (oj >= 0 && (bj < 0 || ow > bw || (ow == bw && oj < bj))) { bw = ow; bj = oj; }
                }
                next = bj;
                ++fb;
            }
            if (lane == 0) {
                tabu[next >> 5] |= 1u << (next & 31);
                tour[step] = next;
            }
            __syncwarp();
            cur = next;
        }
        if (lane == 0) {
            tour[n] = start;
            if (fb) atomicAdd(p.argmax_fallbacks, fb);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Data-parallel "independent roulette" (select_next_data_parallel,
// construction.hpp:129-162; the paper's Fig. 1): city j scores w_j * u_j with
// its own draw (draw index j), the winner is the lowest-index maximum over
// the unvisited cities (tile reduction order does not change it), and a
// non-positive best falls back to the lowest unvisited city.
__global__ void __launch_bounds__(128) k_construct_data_parallel(ConstructParams p) {
    extern __shared__ uint32_t smem_tabu[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* tabu = smem_tabu + wib * p.tabu_words;
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
            for (int j = lane; j < n; j += 32) {
                if (tabu_test(tabu, j)) continue;
                const double u = philox_uniform(p.seed, p.iteration, kg,
                                                static_cast<uint32_t>(step), static_cast<uint32_t>(j));
                const double s = row[j] * u;
                if (bj < 0 || s > bs) { bs = s; bj = j; }
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
