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
// Roulette over the full row.  NV = 128-bit loads per lane per round,
// C = NV*V cities per lane per round, MAXR = max rounds (R <= MAXR).
template <typename WT, int NV, int MAXR>
__global__ void __launch_bounds__(32, 16) k_construct_roulette(ConstructParams p) {
    using VT = typename VecOf<WT>::T;
    constexpr int V = VecOf<WT>::V;
    constexpr int C = NV * V;
    constexpr int NWIN = (C + 31) / 32;
    constexpr int D1 = ceil_log2<C>();
    constexpr bool F32 = sizeof(WT) == 4;

    extern __shared__ uint32_t smem_tabu[];
    uint32_t* tabu = smem_tabu;
    const int lane = threadIdx.x & 31;
    const int n = p.n;
    const WT* __restrict__ wbase = static_cast<const WT*>(p.w);

    // Certification constants (see header comment). All bounds are relative
    // to an upper bound Thi of the exact (scaled) total.
    const double rel_ours = (F32 ? (1.0 + D1) * 0x1.0p-24 : D1 * 0x1.0p-53) +
                            (double)(8 + MAXR + C + 8) * 0x1.0p-53;
    const double rel_ref = (double)(n + 2) * 0x1.0p-53 * (1.0 + 0x1.0p-30);
    const double abs_q = F32 ? (double)n * 0x1.0p-149 : 0.0; // 2 * n * 2^-150

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
            const WT* __restrict__ row = wbase + static_cast<size_t>(cur) * p.PW;
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
                    const VT* rv = reinterpret_cast<const VT*>(row + r * 32 * C) + lane;
                    WT x[C];
#pragma unroll
                    for (int t = 0; t < NV; ++t) {
                        const int e0 = t * V;
                        const uint32_t bits = (win[e0 >> 5] >> (e0 & 31)) & ((1u << V) - 1u);
                        VT v;
                        if (bits != (1u << V) - 1u) {
                            v = __ldg(rv + t * 32);
                        } else {
                            if constexpr (F32) v = make_float4(0.f, 0.f, 0.f, 0.f);
                            else v = make_double2(0.0, 0.0);
                        }
                        if constexpr (F32) {
                            x[e0 + 0] = v.x; x[e0 + 1] = v.y; x[e0 + 2] = v.z; x[e0 + 3] = v.w;
                        } else {
                            x[e0 + 0] = v.x; x[e0 + 1] = v.y;
                        }
                    }
#pragma unroll
                    for (int e = 0; e < C; ++e)
                        if ((win[e >> 5] >> (e & 31)) & 1u) x[e] = WT(0);
                    double d = static_cast<double>(tree_sum<WT, C>(x));
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
            const double u = philox_uniform(p.seed, p.iteration, kg, static_cast<uint32_t>(step), 0);
            const double t = u * T;
            bool ok = (T > 0.0) && (T < 1e300);
            int next = -1;
            if (ok) {
                // round holding the crossing
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
                    int jstar = -1;
                    double Pj = 0.0, Pprev = 0.0;
                    if (lane == L) {
                        double acc = base + (L == 0 ? 0.0 : prev_lane);
                        const int cbase = rs * 32 * C + L * C;
                        const int w0 = cbase >> 5, sh = cbase & 31;
                        uint32_t win[NWIN];
#pragma unroll
                        for (int i = 0; i < NWIN; ++i)
                            win[i] = __funnelshift_r(tabu[w0 + i], tabu[w0 + i + 1], sh);
                        const VT* rv = reinterpret_cast<const VT*>(row + rs * 32 * C) + L;
#pragma unroll
                        for (int tt = 0; tt < NV; ++tt) {
                            const VT v = __ldg(rv + tt * 32);
                            WT xs[V];
                            if constexpr (F32) { xs[0] = v.x; xs[1] = v.y; xs[2] = v.z; xs[3] = v.w; }
                            else { xs[0] = v.x; xs[1] = v.y; }
#pragma unroll
                            for (int q = 0; q < V; ++q) {
                                const int e = tt * V + q;
                                if (jstar < 0 && !((win[e >> 5] >> (e & 31)) & 1u)) {
                                    const double na = acc + static_cast<double>(xs[q]);
                                    if (na > t) {
                                        jstar = cbase + e;
                                        Pj = na;
                                        Pprev = acc;
                                    }
                                    acc = na;
                                }
                            }
                        }
                    }
                    jstar = __shfl_sync(kFull, jstar, L);
                    Pj = __shfl_sync(kFull, Pj, L);
                    Pprev = __shfl_sync(kFull, Pprev, L);
                    if (jstar < 0 || jstar >= n) {
                        ok = false;
                    } else {
                        const double Thi = T * (1.0 + 0x1.0p-20) + abs_q;
                        const double E = (rel_ours + rel_ref + 0x1.0p-51) * Thi + abs_q;
                        const double M = 2.0 * E * (1.0 + 0x1.0p-20);
                        ok = (Pj - t > M) && (t - Pprev > M);
                        next = jstar;
                    }
                }
            }
            if (!ok) {
                next = exact_walk(p.w64 + static_cast<size_t>(cur) * p.P64, tabu, n,
                                  p.tabu_words, u, lane);
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
