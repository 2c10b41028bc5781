// Tour-length, iteration-statistics and pheromone-update kernels (sm_100a).
//
//   k_tour_length      tour_length (model.hpp:205-226) as an int64 warp
//                      reduction, w_k = 1.0 / (double)C_k
//                      (inverse_lengths, pheromone.hpp:123-128), and the
//                      per-city successor/predecessor tables the row-gather
//                      deposit reads.
//   k_iter_stats       iteration best (strict <, lowest ant wins ties), the
//                      int64 length sum for the mean, and the best-so-far tour
//                      (engine.hpp:117-129, 151-154).
//   k_evaporate        evaporate (pheromone.hpp:174-189): tau *= (1 - rho),
//                      one IEEE multiply per cell, 128-bit streaming.
//   k_deposit_atomic   deposit_accumulate (pheromone.hpp:195-208) as the
//                      paper's atomic scatter: one thread per (ant, edge),
//                      two red.global.add.f64.  Order-nondeterministic;
//                      parity is 1e-5 relative (measured ~1e-16).
//   k_rows<MODE>       one CTA per pheromone row, fusing
//                        MODE_GATHER: the deterministic scatter-to-gather
//                          deposit (gather_cell family, pheromone.hpp:133-341)
//                          restated in O(m) per row: contributions w_k land in
//                          a shared-memory row in ascending ant order, then
//                          tau = fl(fl(tau * keep) + acc)  (bit-exact, :183 then :220);
//                        MODE_DELTA: tau = fl(fl(tau * keep) + delta) for the
//                          multi-GPU atomic path (delta all-reduced over NCCL);
//                      followed (all modes) by compute_choice_info
//                      (model.hpp:154-173): choice = pow(tau, alpha) *
//                      eta_beta[dist] with the host-libm table, diagonal 0,
//                      and the per-row power-of-two scaled fp32 / permuted
//                      copies the construction kernel streams.
#pragma once

#include <cstdint>

#include "construct.cuh"
#include "libm_pow.cuh"

namespace acob200 {

__global__ void k_tour_length(const int32_t* __restrict__ tours, const int32_t* __restrict__ dist,
                              int n, int P64, int mloc, int64_t* __restrict__ len,
                              double* __restrict__ inv, int32_t* __restrict__ succ,
                              int32_t* __restrict__ pred, int S) {
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    for (int kl = blockIdx.x * warps + (threadIdx.x >> 5); kl < mloc; kl += gridDim.x * warps) {
        const int32_t* t = tours + static_cast<size_t>(kl) * (n + 1);
        long long acc = 0;
        // batches of 8 edges per lane: all (random) distance gathers of a
        // batch in flight together; the succ/pred scatter stores after them
        constexpr int B = 8;
        for (int s0 = lane; s0 < n; s0 += 32 * B) {
            int a[B], b[B], d[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int s = s0 + 32 * u;
                a[u] = s < n ? t[s] : 0;
                b[u] = s < n ? t[s + 1] : 0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u)
                d[u] = s0 + 32 * u < n ? __ldg(dist + static_cast<size_t>(a[u]) * P64 + b[u]) : 0;
            if (succ) {
#pragma unroll
                for (int u = 0; u < B; ++u)
                    if (s0 + 32 * u < n) {
                        succ[static_cast<size_t>(a[u]) * S + kl] = b[u];
                        pred[static_cast<size_t>(b[u]) * S + kl] = a[u];
                    }
            }
#pragma unroll
            for (int u = 0; u < B; ++u) acc += d[u];
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
        if (lane == 0) {
            len[kl] = acc;
            inv[kl] = 1.0 / static_cast<double>(acc);
        }
    }
}

// Debug-mode tour validation (aco_gpu_params::validate_tours): the checks
// the reference makes on every tour before depositing — TourBuffer::make
// (pheromone.hpp:67-90) recomputes tour_length (model.hpp:205-226), which
// throws not_closed if tour[n] != tour[0], not_a_permutation if a city is
// out of range or repeated, and the buffer then throws inconsistent_length if
// the stored length differs.  One warp per ant with the ant's visited bitset
// in shared memory; the first failure in (ant, check) order wins, as the
// reference's ascending ant loop throws at the first one:
// err = min over failing ants of (ant << 2) | code, code 1 not_closed,
// 2 not_a_permutation, 3 inconsistent_length.
__global__ void k_validate_tours(const int32_t* __restrict__ tours, const int32_t* __restrict__ dist,
                                 const int64_t* __restrict__ len, int n, int P64, int mloc,
                                 unsigned long long* __restrict__ err) {
    extern __shared__ uint32_t seen_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int words = (n + 31) >> 5;
    uint32_t* seen = seen_all + wib * words;
    const int warps = blockDim.x >> 5;
    for (int kl = blockIdx.x * warps + wib; kl < mloc; kl += gridDim.x * warps) {
        const int32_t* t = tours + static_cast<size_t>(kl) * (n + 1);
        for (int w = lane; w < words; w += 32) seen[w] = 0u;
        __syncwarp();
        unsigned long long code = 0;
        if (t[n] != t[0]) code = 1;
        bool dup = false;
        long long acc = 0;
        for (int s = lane; s < n; s += 32) {
            const int c = t[s];
            if (c < 0 || c >= n) {
                dup = true;
                continue;
            }
            const uint32_t bit = 1u << (c & 31);
            if (atomicOr(seen + (c >> 5), bit) & bit) dup = true;
            const int d = t[s + 1];
            if (d >= 0 && d < n) acc += __ldg(dist + static_cast<size_t>(c) * P64 + d);
        }
        dup = __any_sync(kFull, dup);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
        if (code == 0 && dup) code = 2;
        if (code == 0 && acc != len[kl]) code = 3;
        if (lane == 0 && code) atomicMin(err, (static_cast<unsigned long long>(kl) << 2) | code);
        __syncwarp();
    }
}

// One CTA.  stats[0] = best length, stats[1] = best local ant, stats[2] =
// length sum.  Copies the best tour when it strictly improves best_so_far.
__global__ void __launch_bounds__(1024) k_iter_stats(const int64_t* __restrict__ len, int mloc,
                                                     const int32_t* __restrict__ tours, int n,
                                                     long long* __restrict__ stats,
                                                     long long* __restrict__ best_so_far,
                                                     int32_t* __restrict__ best_tour,
                                                     int update_best) {
    __shared__ long long s_len[32], s_sum[32];
    __shared__ int s_idx[32];
    __shared__ int s_improved, s_best;
    long long bl = LLONG_MAX, sum = 0;
    int bi = INT_MAX;
    for (int k = threadIdx.x; k < mloc; k += blockDim.x) {
        const long long l = len[k];
        sum += l;
        if (l < bl) { bl = l; bi = k; } // k ascending per thread: first wins
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const long long ol = __shfl_xor_sync(kFull, bl, off);
        const int oi = __shfl_xor_sync(kFull, bi, off);
        sum += __shfl_xor_sync(kFull, sum, off);
        if (ol < bl || (ol == bl && oi < bi)) { bl = ol; bi = oi; }
    }
    if (lane == 0) { s_len[w] = bl; s_idx[w] = bi; s_sum[w] = sum; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        bl = lane < nw ? s_len[lane] : LLONG_MAX;
        bi = lane < nw ? s_idx[lane] : INT_MAX;
        sum = lane < nw ? s_sum[lane] : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const long long ol = __shfl_xor_sync(kFull, bl, off);
            const int oi = __shfl_xor_sync(kFull, bi, off);
            sum += __shfl_xor_sync(kFull, sum, off);
            if (ol < bl || (ol == bl && oi < bi)) { bl = ol; bi = oi; }
        }
        if (lane == 0) {
            stats[0] = bl;
            stats[1] = bi;
            stats[2] = sum;
            const int imp = update_best && bl < *best_so_far;
            if (imp) *best_so_far = bl;
            s_improved = imp;
            s_best = bi;
        }
    }
    __syncthreads();
    if (s_improved) {
        const int32_t* src = tours + static_cast<size_t>(s_best) * (n + 1);
        for (int s = threadIdx.x; s <= n; s += blockDim.x) best_tour[s] = src[s];
    }
}

// Sharded statistics entirely on the device (no host round trip between
// the construction and the update).  Stage 1, before the MIN / SUM
// all-reduces: with shift > 0, key = (best length << shift) | global ant, so
// the MIN gives the iteration best AND its lowest global ant (engine.hpp:
// 117-129 tie rule) in one collective — the host picks shift so that every
// possible length fits (n * max_d < 2^(62 - shift)); with shift == 0 the key
// is the length alone and k_shard_ant + a second MIN resolve the ant.
__global__ void k_shard_key(long long* stats, int ant_begin, int mloc, int shift) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        stats[4] = mloc <= 0 ? LLONG_MAX
                   : shift > 0 ? (stats[0] << shift) | static_cast<long long>(ant_begin + stats[1])
                               : stats[0];
        stats[6] = stats[2];
    }
}
// Two-stage key, after the length MIN: this rank's candidate ant if its own
// best equals the global best, else +inf (then all-reduce MIN).
__global__ void k_shard_ant(long long* stats, int ant_begin, int mloc) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        stats[5] = (mloc > 0 && stats[0] == stats[4]) ? static_cast<long long>(ant_begin + stats[1])
                                                      : LLONG_MAX;
}
__device__ __forceinline__ long long shard_best_len(const long long* stats, int shift) {
    return shift > 0 ? stats[4] >> shift : stats[4];
}
__device__ __forceinline__ long long shard_best_ant(const long long* stats, int shift) {
    if (stats[4] == LLONG_MAX) return -1;
    return shift > 0 ? (stats[4] & ((1LL << shift) - 1)) : stats[5];
}
// Stage 2, after them: the rank owning the winning ant copies its tour into
// the exchange buffer, the others zero it; an all-reduce MAX replicates it
// (tour entries are >= 0).
__global__ void k_owner_tour(const long long* __restrict__ stats, const int32_t* __restrict__ tours,
                             int n, int ant_begin, int ant_end, int32_t* __restrict__ tourbuf,
                             int shift) {
    const long long ant = shard_best_ant(stats, shift);
    const bool own = ant >= ant_begin && ant < ant_end;
    const int32_t* src = tours + static_cast<size_t>(own ? ant - ant_begin : 0) * (n + 1);
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s <= n; s += gridDim.x * blockDim.x)
        tourbuf[s] = own ? src[s] : 0;
}
// Stage 3: best-so-far and its tour on strict improvement (engine.hpp:151-154).
__global__ void __launch_bounds__(1024) k_best_update(long long* stats, const int32_t* __restrict__ tourbuf,
                                                      int n, int32_t* __restrict__ best_tour, int shift) {
    __shared__ int imp;
    const long long gl = shard_best_len(stats, shift);
    if (threadIdx.x == 0) imp = gl < stats[3];
    __syncthreads();
    if (imp)
        for (int s = threadIdx.x; s <= n; s += blockDim.x) best_tour[s] = tourbuf[s];
    __syncthreads();
    if (threadIdx.x == 0 && imp) stats[3] = gl;
}

__global__ void k_evaporate(double* __restrict__ tau, size_t count2, double keep) {
    double2* t2 = reinterpret_cast<double2*>(tau);
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count2;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double2 v = t2[i];
        v.x = __dmul_rn(v.x, keep);
        v.y = __dmul_rn(v.y, keep);
        t2[i] = v;
    }
}

// Multi-GPU atomic path, NCCL wire in fp32: the local fp64 delta (summed
// by red.f64) is rounded once to fp32 for the all-reduce and zeroed for the
// next iteration.  Half the exchange bytes; the rounding (2^-24 relative,
// plus the G-term fp32 sum inside NCCL) stays far inside the path's 1e-5
// relative tau tolerance, and every rank receives the same reduced value.
__global__ void k_delta_pack(double* __restrict__ delta, float* __restrict__ d32, size_t count2) {
    double2* d2 = reinterpret_cast<double2*>(delta);
    float2* f2 = reinterpret_cast<float2*>(d32);
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count2;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double2 v = d2[i];
        f2[i] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
        d2[i] = make_double2(0.0, 0.0);
    }
}

// One thread per (ant, step); edges (t[s], t[s+1]) and the mirror.
__global__ void k_deposit_atomic(const int32_t* __restrict__ tours, const double* __restrict__ inv,
                                 int n, int P64, int mloc, double* __restrict__ target) {
    const size_t total = static_cast<size_t>(mloc) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int kl = static_cast<int>(i / n), s = static_cast<int>(i - static_cast<size_t>(kl) * n);
        const int32_t* t = tours + static_cast<size_t>(kl) * (n + 1);
        const int a = t[s], b = t[s + 1];
        const double w = inv[kl];
        atomicAdd(target + static_cast<size_t>(a) * P64 + b, w);
        atomicAdd(target + static_cast<size_t>(b) * P64 + a, w);
    }
}

// Symmetric accumulate deposit (one-GPU roulette / data-parallel): the
// reference adds w_k to tau[a][b] AND tau[b][a] (pheromone.hpp:198-205), two
// equal sums, so one red per edge into the upper-triangle cell of a cleared
// delta carries both; k_rows<MODE_DELTA_SYM> applies it to both cells after
// the evaporation (the atomic path's 1e-5 relative contract: the same sums,
// associated differently).
__global__ void k_deposit_sym(const int32_t* __restrict__ tours, const double* __restrict__ inv,
                              int n, int P64, int mloc, double* __restrict__ delta) {
    const size_t total = static_cast<size_t>(mloc) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int kl = static_cast<int>(i / n), s = static_cast<int>(i - static_cast<size_t>(kl) * n);
        const int32_t* t = tours + static_cast<size_t>(kl) * (n + 1);
        const int a = t[s], b = t[s + 1];
        atomicAdd(delta + static_cast<size_t>(min(a, b)) * P64 + max(a, b), inv[kl]);
    }
}

// Accumulate deposit for the nn selection (config 5).  An edge a -> b whose
// head is member q of a's nn list (the construction recorded q) adds w_k to
// the compact slot dnn[a][q] — n x nn doubles, 2.4 MB at 10k, L2-resident —
// instead of two reds scattered over the 800 MB tau; every other edge (argmax
// fallbacks, the closing edge) reds into tau directly.  k_apply_nn then adds
// each slot to tau[a][b] AND tau[b][a] (the reference deposits w_k on both,
// pheromone.hpp:198-205) and clears it.  Same sums as deposit_accumulate in
// a different order: the atomic path's 1e-5 relative contract.
__global__ void k_deposit_nn(const int32_t* __restrict__ tours, const uint8_t* __restrict__ qpos,
                             const double* __restrict__ inv, int n, int P64, int mloc, int nn,
                             double* __restrict__ dnn, double* __restrict__ tau) {
    const size_t total = static_cast<size_t>(mloc) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int kl = static_cast<int>(i / n), s = static_cast<int>(i - static_cast<size_t>(kl) * n);
        const int32_t* t = tours + static_cast<size_t>(kl) * (n + 1);
        const int a = t[s];
        const int q = qpos[i];
        const double w = inv[kl];
        if (q < nn) {
            atomicAdd(dnn + static_cast<size_t>(a) * nn + q, w);
        } else {
            const int b = t[s + 1];
            atomicAdd(tau + static_cast<size_t>(a) * P64 + b, w);
            atomicAdd(tau + static_cast<size_t>(b) * P64 + a, w);
        }
    }
}

__global__ void k_apply_nn(double* __restrict__ dnn, const int32_t* __restrict__ nn_lists, int n,
                           int nn, int P64, double* __restrict__ tau) {
    const size_t slots = static_cast<size_t>(n) * nn;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < slots;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double d = dnn[i];
        if (d != 0.0) {
            const int a = static_cast<int>(i / nn), b = nn_lists[i];
            atomicAdd(tau + static_cast<size_t>(a) * P64 + b, d);
            atomicAdd(tau + static_cast<size_t>(b) * P64 + a, d);
            dnn[i] = 0.0;
        }
    }
}

// ---- fixed-point accumulate (ACO_WIRE_FIXED64 / ACO_WIRE_MULTIMEM) -------
// Every deposit w_k = 1/C_k is added as the integer round(w_k * 2^s) with
// 64-bit integer reds, so each cell's delta is an EXACT integer sum: the
// result does not depend on the order of the reds, on the number of GPUs or
// on how an all-reduce (ncclInt64) or the NVSwitch (multimem) combines them
// — tau is bit-identical on every rank and for every G.  s is chosen per
// iteration from the colony's best length L (k_fixed_scale): no cell can
// receive more than sum_k w_k <= m / L (an edge is used at most twice per
// tour), so with S = 2m/L < 2^(e+1), s = 60 - e keeps every sum below 2^61.
// Per contribution the rounding is <= 2^-(s+1), i.e. relative <= m * (C_max /
// C_min) * 2^-61 ~ 1e-14 at 10^4 ants — far inside the atomic path's 1e-5
// relative contract (pheromone.hpp:195-208, deposit_accumulate).
// stats[7] receives s (or -1: a zero-length tour, 1/C_k = inf, which no
// fixed-point scale represents — the engine then fails the iteration).
__global__ void k_fixed_scale(long long* stats, int m, int shard_shift, int sharded) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const long long L = sharded ? shard_best_len(stats, shard_shift) : stats[0];
    if (L <= 0) {
        stats[7] = -1;
        return;
    }
    const double S = 2.0 * static_cast<double>(m) / static_cast<double>(L);
    stats[7] = 60 - ilogb(S);
}

template <bool MULTIMEM>
__device__ __forceinline__ void red_u64(unsigned long long* addr, unsigned long long v) {
    if constexpr (MULTIMEM) {
        // NVLS: one red to the multicast address, applied by the NVSwitch to
        // the delta of every GPU bound to the object
        asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(addr), "l"(v) : "memory");
    } else {
        atomicAdd(addr, v);
    }
}

template <bool MULTIMEM>
__global__ void k_deposit_fixed(const int32_t* __restrict__ tours, const double* __restrict__ inv,
                                int n, int P64, int mloc, const long long* __restrict__ stats,
                                unsigned long long* __restrict__ target) {
    const int sh = static_cast<int>(stats[7]);
    if (sh < 0) return;
    const size_t total = static_cast<size_t>(mloc) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int kl = static_cast<int>(i / n), s = static_cast<int>(i - static_cast<size_t>(kl) * n);
        const int32_t* t = tours + static_cast<size_t>(kl) * (n + 1);
        const int a = t[s], b = t[s + 1];
        const unsigned long long v = __double2ull_rn(scalbn(inv[kl], sh));
        red_u64<MULTIMEM>(target + static_cast<size_t>(a) * P64 + b, v);
        red_u64<MULTIMEM>(target + static_cast<size_t>(b) * P64 + a, v);
    }
}

// nn selection with the fixed-point accumulate (config 5, any G): list edges
// add round(w_k 2^s) to the compact int64 slots dnn[a][q]; every other edge
// (argmax fallbacks, the closing edge) is appended to a record list
// {a, b, round(w_k 2^s)}.  Sharded, only the compact slots (n x nn x 8 B,
// 2.4 MB at 10k) are all-reduced and the records all-gathered — instead of
// the n^2 delta (800 MB) — and every rank scatters the same integers into its
// local dense delta (k_apply_nn_fixed, k_apply_records): exact sums, so tau is
// bit-identical on every rank and for every G.
struct __align__(16) DepositRecord {
    int32_t a, b;
    unsigned long long v;
};

__global__ void k_deposit_nn_fixed(const int32_t* __restrict__ tours, const uint8_t* __restrict__ qpos,
                                   const double* __restrict__ inv, int n, int mloc, int nn,
                                   const long long* __restrict__ stats,
                                   unsigned long long* __restrict__ dnn, DepositRecord* __restrict__ rec,
                                   unsigned long long* __restrict__ rec_count) {
    const int sh = static_cast<int>(stats[7]);
    if (sh < 0) return;
    const size_t total = static_cast<size_t>(mloc) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int kl = static_cast<int>(i / n), s = static_cast<int>(i - static_cast<size_t>(kl) * n);
        const int32_t* t = tours + static_cast<size_t>(kl) * (n + 1);
        const int a = t[s];
        const int q = qpos[i];
        const unsigned long long v = __double2ull_rn(scalbn(inv[kl], sh));
        if (q < nn) {
            atomicAdd(dnn + static_cast<size_t>(a) * nn + q, v);
        } else {
            const unsigned long long at = atomicAdd(rec_count, 1ull);
            rec[at] = DepositRecord{a, t[s + 1], v};
        }
    }
}

__global__ void k_apply_nn_fixed(unsigned long long* __restrict__ dnn, const int32_t* __restrict__ nn_lists,
                                 int n, int nn, int P64, unsigned long long* __restrict__ delta) {
    const size_t slots = static_cast<size_t>(n) * nn;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < slots;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const unsigned long long d = dnn[i];
        if (d != 0ull) {
            const int a = static_cast<int>(i / nn), b = nn_lists[i];
            atomicAdd(delta + static_cast<size_t>(a) * P64 + b, d);
            atomicAdd(delta + static_cast<size_t>(b) * P64 + a, d);
            dnn[i] = 0ull;
        }
    }
}

// records of `shards` ranks, rank g's at rec[g * stride], counts[g] of them
__global__ void k_apply_records(const DepositRecord* __restrict__ rec, const unsigned long long* __restrict__ counts,
                                int shards, size_t stride, int P64, unsigned long long* __restrict__ delta) {
    for (int g = 0; g < shards; ++g) {
        const size_t cnt = counts[g];
        const DepositRecord* r = rec + static_cast<size_t>(g) * stride;
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cnt;
             i += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const DepositRecord e = r[i];
            atomicAdd(delta + static_cast<size_t>(e.a) * P64 + e.b, e.v);
            atomicAdd(delta + static_cast<size_t>(e.b) * P64 + e.a, e.v);
        }
    }
}

// Cross-GPU barrier over the multicast object (ACO_WIRE_MULTIMEM), one
// thread: make this GPU's reds visible system-wide, add 1 to every GPU's copy
// of the flag with one release red through the switch, then wait until the
// local copy shows all `world` arrivals of this epoch.
__global__ void k_mc_barrier(unsigned long long* mc_flag, const unsigned long long* uc_flag,
                             unsigned long long target) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc_flag), "l"(1ull) : "memory");
    unsigned long long v = 0;
    do {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(uc_flag) : "memory");
    } while (v < target);
}

// MODE_DELTA32: MODE_DELTA reading the fp32 all-reduced delta (NCCL fp32
// wire; k_delta_pack already zeroed the fp64 delta)
// MODE_DELTA_FIX: tau = fl(fl(tau*keep) + delta_i64 * 2^-s) from the exact
// fixed-point sums (k_deposit_fixed), then clears the delta.
#ifndef ACO_SYM_DEPOSIT
#define ACO_SYM_DEPOSIT 1 // one-GPU accumulate through the symmetric upper-triangle delta
#endif
// MODE_DELTA_SYM: MODE_DELTA over a symmetric delta kept in the upper
// triangle only (k_deposit_sym: one red per edge instead of two): row i reads
// delta[i][j] for j > i and the column delta[j][i] for j < i; the buffer is
// cleared before the deposit (a cell is read by two rows, so no row can clear it)
enum { MODE_CHOICE = 0, MODE_GATHER = 1, MODE_DELTA = 2, MODE_DELTA32 = 3, MODE_DELTA_FIX = 4,
       MODE_DELTA_SYM = 5 };

struct RowParams {
    double* tau;             // n x P64
    double* choice64;        // n x P64
    float* choice32;         // n x PW (fp32 stream) or null
    double* choice_perm64;   // n x PW (fp64 stream) or null
    int32_t* scale_exp;      // n
    const int32_t* dist;     // n x P64
    const double* lut;       // eta^beta by distance, or null
    const double* etab;      // n x P64 eta^beta, or null
    double* delta;           // MODE_DELTA: n x P64
    const float* delta32;    // MODE_DELTA32: n x P64
    const int32_t* succ;     // MODE_GATHER: [shard][city][S]
    const int32_t* pred;
    const double* inv;       // [shard][S]
    const int32_t* nn_lists; // n x nn (nn selection) or null
    double* choice_nn;       // n x nn: choice64[i][nn_lists[i][q]] (nn selection)
    int2* choice_nn32;       // n x nn records {city id, fp32 bits of the weight scaled by 2^nn_scale[i]} (row max -> [2^kScaleExp, 2^(kScaleExp+1))): one 8-byte load per member in the nn fast path
    int32_t* nn_scale;       // n
    int nn;
    int n, P64, PW, C, V, LA;
    int shards, S, m;        // ants: shard g holds global ants [g*S, min(m,(g+1)*S))
    double alpha, keep;
    const LibmPowTables* powtab; // host libm's pow tables (alpha not in {0, 1})
    unsigned long long* delta_fix; // MODE_DELTA_FIX: n x P64 fixed-point sums
    const long long* stats;        // MODE_DELTA_FIX: stats[7] = the scale exponent s
    int row_begin, row_end;        // k_rows_gather_warp: the rows this launch folds
    int nat;                       // streamed rows in the natural layout (RowLayout)
};

// Write one row of the permuted streamed layout (stream_pos) from the natural
// row in shared memory: one V-wide vector slot (V consecutive cities of one
// lane chunk, or a pad slot) per iteration, so the index arithmetic is two
// divisions per vector instead of three per city.  V = 4: fp32 scaled by
// 2^sc; V = 2: fp64 as is.
template <int V, typename OT>
__device__ __forceinline__ void write_stream_row(OT* __restrict__ crow, const double* rowbuf, int n,
                                                 int PW, int C, int LA, int sc, int tid,
                                                 int nthreads, bool nat) {
    const int LP = LA + kPad, NVL = C / V, RS = LP * NVL; // vector slots per round
    nat = nat && (NVL & 1) != 0; // natural layout (RowLayout, odd NV)
    const int nslots = PW / V;
    for (int s = tid; s < nslots; s += nthreads) {
        int l = 0, c0 = s * V;
        if (!nat) {
            const int r = s / RS, rem = s - r * RS;
            const int t = rem / LP;
            l = rem - t * LP;
            c0 = r * LA * C + l * C + t * V;
        }
        if constexpr (V == 4) {
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
            if (l < LA) {
                if (c0 + 0 < n) o.x = __double2float_rn(scalbn(rowbuf[c0 + 0], sc));
                if (c0 + 1 < n) o.y = __double2float_rn(scalbn(rowbuf[c0 + 1], sc));
                if (c0 + 2 < n) o.z = __double2float_rn(scalbn(rowbuf[c0 + 2], sc));
                if (c0 + 3 < n) o.w = __double2float_rn(scalbn(rowbuf[c0 + 3], sc));
            }
            reinterpret_cast<float4*>(crow)[s] = o;
        } else {
            double2 o = make_double2(0.0, 0.0);
            if (l < LA) {
                if (c0 + 0 < n) o.x = rowbuf[c0 + 0];
                if (c0 + 1 < n) o.y = rowbuf[c0 + 1];
            }
            reinterpret_cast<double2*>(crow)[s] = o;
        }
    }
}

// Exponent the streamed fp32 copies scale each row's maximum to: the max
// lands in [2^kScaleExp, 2^(kScaleExp+1)), so a sum of up to 2^15 weights
// stays below FLT_MAX (2^128) while small weights keep as many bits as
// possible before becoming subnormal (a subnormal weight only costs the
// certification its absolute 2^-150 term).
constexpr int kScaleExp = 112;

// Row i's nn list weights (one warp, lanes = members; nn <= 32 for the
// fp32 copy): fp64 for the exact paths, and an fp32 copy scaled by the
// exact power of two that puts the list maximum in [2^112, 2^113) for the
// nn fast path's fp32 scan (a scaled weight below 2^-126 only loses
// absolute precision, <= 2^-150 each, which the certification counts).
__device__ __forceinline__ void write_nn_row(const RowParams& p, const double* src, int i, int lane) {
    const size_t base = static_cast<size_t>(i) * p.nn;
    double w = 0.0;
    if (lane < p.nn) {
        w = src[p.nn_lists[base + lane]];
        p.choice_nn[base + lane] = w;
    }
    for (int q = lane + 32; q < p.nn; q += 32) p.choice_nn[base + q] = src[p.nn_lists[base + q]];
    if (p.choice_nn32 && p.nn <= 32) {
        double mx = w;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, off));
        const int sc = mx > 0.0 ? kScaleExp - ilogb(mx) : 0;
        if (lane < p.nn)
            p.choice_nn32[base + lane] =
                make_int2(p.nn_lists[base + lane], __float_as_int(__double2float_rn(scalbn(w, sc))));
        if (lane == 0) p.nn_scale[i] = sc;
    }
}

__device__ __forceinline__ double tau_pow(double t, double alpha, const LibmPowTables* powtab) {
    if (alpha == 1.0) return t;  // pow(x, 1) == x exactly (SURVEY [E1])
    if (alpha == 0.0) return 1.0; // pow(x, 0) == 1 exactly
    return libm_pow(t, alpha, powtab); // the host glibc pow, replayed (libm_pow.cuh)
}

// One CTA (256 threads) per row.  The elementwise pass works on column PAIRS
// (16-byte tau / choice / delta accesses, 8-byte dist) in batches of EB pairs
// per thread, all loads of a batch issued before any eta^beta gather and all
// gathers before the arithmetic, so each thread keeps 3*EB independent memory
// requests in flight.  Pad columns (n <= j < P64) compute 0 (tau pad = 0) and
// are written like the others.  The shared row (P64 doubles) is used only
// when something needs the finished row: the gather fold, the permuted
// streamed copies (row max first) and the nn weights; otherwise the kernel
// runs with no dynamic shared memory and full occupancy.
// CTAs per SM the register budget must allow: 4 for the choice pass (the
// one-GPU update: pr2392 -3%, 10k -5.5%, 64 registers), 3 for the others
// (the delta pass at 64 registers was 9% slower)
template <int MODE>
__global__ void __launch_bounds__(256, MODE == MODE_CHOICE ? 4 : 3) k_rows(RowParams p) {
    extern __shared__ double rowbuf[]; // P64 doubles when use_row
    __shared__ double s_max[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = p.n;
    const bool use_row = MODE == MODE_GATHER || p.choice32 || p.choice_perm64;
    const bool need_sync = use_row || p.choice_nn;
    const int n2 = p.P64 >> 1;
    constexpr int EB = MODE == MODE_CHOICE ? 4 : 3;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        double* trow = p.tau + static_cast<size_t>(i) * p.P64;
        if constexpr (MODE == MODE_GATHER) {
            for (int j = tid; j < p.P64; j += blockDim.x) rowbuf[j] = 0.0;
            __syncthreads();
            // Contributions to column c arrive in ascending global ant order
            // (shards are contiguous ant ranges); warp `warp` owns columns
            // c % 8 == warp so its shared-memory updates never race.  Within
            // a chunk of 16 ants the 32 lanes carry (ant a = lane/2, pred or
            // succ); equal columns are folded in lane (= ant) order.
            for (int g = 0; g < p.shards; ++g) {
                const int kbeg = g * p.S;
                const int cnt = min(p.S, p.m - kbeg);
                const int32_t* sc = p.succ + (static_cast<size_t>(g) * n + i) * p.S;
                const int32_t* pc = p.pred + (static_cast<size_t>(g) * n + i) * p.S;
                const double* wv = p.inv + static_cast<size_t>(g) * p.S;
                for (int k0 = 0; k0 < cnt; k0 += 16) {
                    const int k = k0 + (lane >> 1);
                    int col = -1;
                    double w = 0.0;
                    if (k < cnt) {
                        col = (lane & 1) ? sc[k] : pc[k];
                        w = wv[k];
                    }
                    const bool mine = col >= 0 && (col & 7) == warp;
                    const unsigned mm = __ballot_sync(kFull, mine);
                    if (mine) {
                        const unsigned grp = __match_any_sync(mm, col);
                        double acc = rowbuf[col];
                        for (unsigned b = grp; b; b &= b - 1) acc += __shfl_sync(grp, w, __ffs(b) - 1);
                        if (lane == __ffs(grp) - 1) rowbuf[col] = acc;
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
        }
        double mx = 0.0;
        const int2* drow2 = reinterpret_cast<const int2*>(p.dist + static_cast<size_t>(i) * p.P64);
        const double2* erow2 =
            p.etab ? reinterpret_cast<const double2*>(p.etab + static_cast<size_t>(i) * p.P64) : nullptr;
        double2* trow2 = reinterpret_cast<double2*>(trow);
        double2* crow2 = reinterpret_cast<double2*>(p.choice64 + static_cast<size_t>(i) * p.P64);
        double2* drw2 = (MODE == MODE_DELTA || MODE == MODE_DELTA_SYM)
                            ? reinterpret_cast<double2*>(p.delta + static_cast<size_t>(i) * p.P64)
                            : nullptr;
        ulonglong2* dfx2 = MODE == MODE_DELTA_FIX
                               ? reinterpret_cast<ulonglong2*>(p.delta_fix + static_cast<size_t>(i) * p.P64)
                               : nullptr;
        const int fsh = MODE == MODE_DELTA_FIX ? static_cast<int>(p.stats[7]) : 0;
        for (int b0 = tid; b0 < n2; b0 += 256 * EB) {
            double2 tv[EB], dl[EB], eb[EB];
            int2 dv[EB];
#pragma unroll
            for (int u = 0; u < EB; ++u) {
                const int j2 = b0 + 256 * u;
                const bool in = j2 < n2;
                tv[u] = in ? trow2[j2] : make_double2(0.0, 0.0);
                dv[u] = (in && !erow2) ? __ldg(drow2 + j2) : make_int2(0, 0);
                if constexpr (MODE == MODE_DELTA) dl[u] = in ? drw2[j2] : make_double2(0.0, 0.0);
                if constexpr (MODE == MODE_DELTA_SYM) {
                    const int j = 2 * j2;
                    const double2 up = (in && j + 1 > i) ? drw2[j2] : make_double2(0.0, 0.0);
                    const double lx = (in && j < i) ? p.delta[static_cast<size_t>(j) * p.P64 + i] : 0.0;
                    const double ly = (in && j + 1 < i) ? p.delta[static_cast<size_t>(j + 1) * p.P64 + i] : 0.0;
                    dl[u] = make_double2(j < i ? lx : (j > i ? up.x : 0.0),
                                         j + 1 < i ? ly : (j + 1 > i ? up.y : 0.0));
                }
                if constexpr (MODE == MODE_DELTA_FIX) {
                    const ulonglong2 f = in ? dfx2[j2] : make_ulonglong2(0ull, 0ull);
                    // exact integer sum -> double (one rounding) -> exact 2^-s scaling
                    dl[u] = make_double2(scalbn(__ull2double_rn(f.x), -fsh), scalbn(__ull2double_rn(f.y), -fsh));
                }
                if constexpr (MODE == MODE_DELTA32) {
                    const float2 f = in ? reinterpret_cast<const float2*>(
                                              p.delta32 + static_cast<size_t>(i) * p.P64)[j2]
                                        : make_float2(0.f, 0.f);
                    dl[u] = make_double2(f.x, f.y);
                }
                if constexpr (MODE == MODE_GATHER) {
                    dl[u] = in ? reinterpret_cast<const double2*>(rowbuf)[j2] : make_double2(0.0, 0.0);
                }
            }
#pragma unroll
            for (int u = 0; u < EB; ++u) {
                const int j2 = b0 + 256 * u;
                if (j2 < n2) {
                    eb[u] = erow2 ? __ldg(erow2 + j2)
                                  : make_double2(__ldg(p.lut + dv[u].x), __ldg(p.lut + dv[u].y));
                }
            }
#pragma unroll
            for (int u = 0; u < EB; ++u) {
                const int j2 = b0 + 256 * u;
                if (j2 < n2) {
                    const int j = 2 * j2;
                    double2 t = tv[u];
                    if constexpr (MODE == MODE_GATHER || MODE == MODE_DELTA || MODE == MODE_DELTA32 ||
                                  MODE == MODE_DELTA_FIX || MODE == MODE_DELTA_SYM) {
                        // pheromone.hpp:183 (evaporate) then :220 / the summed delta
                        t.x = __dadd_rn(__dmul_rn(t.x, p.keep), dl[u].x);
                        t.y = __dadd_rn(__dmul_rn(t.y, p.keep), dl[u].y);
                        trow2[j2] = t;
                        if constexpr (MODE == MODE_DELTA) drw2[j2] = make_double2(0.0, 0.0);
                        if constexpr (MODE == MODE_DELTA_FIX) dfx2[j2] = make_ulonglong2(0ull, 0ull);
                    }
                    double2 c;
                    c.x = (j == i) ? 0.0 : __dmul_rn(tau_pow(t.x, p.alpha, p.powtab), eb[u].x);
                    c.y = (j + 1 == i) ? 0.0 : __dmul_rn(tau_pow(t.y, p.alpha, p.powtab), eb[u].y);
                    crow2[j2] = c;
                    if (use_row) reinterpret_cast<double2*>(rowbuf)[j2] = c;
                    mx = fmax(mx, fmax(c.x, c.y));
                }
            }
        }
        if (p.choice32 || p.choice_perm64) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, off));
            if (lane == 0) s_max[warp] = mx;
        }
        if (need_sync) __syncthreads(); // also orders this block's choice64 stores
        if (p.choice_nn && warp == 0) { // the nn list's weights, contiguous per row (L2-resident)
            const double* src = use_row ? rowbuf : p.choice64 + static_cast<size_t>(i) * p.P64;
            write_nn_row(p, src, i, lane);
        }
        if (p.choice32) {
            double rmx = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) rmx = fmax(rmx, s_max[w]);
            // Exact power-of-two scale: row max -> [2^kScaleExp, 2^(kScaleExp+1)).
            const int sc = rmx > 0.0 ? kScaleExp - ilogb(rmx) : 0;
            if (tid == 0) p.scale_exp[i] = sc;
            write_stream_row<4>(p.choice32 + static_cast<size_t>(i) * p.PW, rowbuf, n, p.PW, p.C,
                                p.LA, sc, tid, blockDim.x, p.nat != 0); // pads 0
        }
        if (p.choice_perm64) {
            write_stream_row<2>(p.choice_perm64 + static_cast<size_t>(i) * p.PW, rowbuf, n, p.PW,
                                p.C, p.LA, 0, tid, blockDim.x, p.nat != 0);
        }
        if (need_sync) __syncthreads();
    }
}

// MODE_GATHER with one WARP per pheromone row (n small enough that a row of
// doubles fits a warp's shared-memory slice).  The CTA-per-row k_rows<GATHER>
// makes each of its 8 warps read the whole contribution stream of the row
// (warp w owns columns c % 8 == w); here one warp reads it once, in
// ascending global ant order, 16 ants (32 contributions: pred, succ) per
// chunk, eight chunks loaded ahead.  Each chunk's (column, weight) pairs are
// staged in shared memory; every lane folds the staged weights of its own
// column in lane (= ant) order starting from the column's running value,
// and the lowest lane holding that column writes it back — so every column
// is the same sequential fold from 0.0 as gather_cell (pheromone.hpp:133-148).
// (A __match_any_sync grouping was 9% slower.)  The
// epilogue (tau update, choice, scaled fp32 stream) is k_rows' own, per warp.
struct __align__(16) StageEntry {
    int col;
    int pad;
    double w;
};
#ifndef ACO_GATHER_AHEAD
#define ACO_GATHER_AHEAD 8 // 16-ant chunks whose contributions are loaded together
#endif
// EPI = false: fold only — the row's ordered sums go to p.delta (row i) and
// k_rows<MODE_DELTA> applies tau = fl(fl(tau*keep) + delta) (the same two
// roundings) and the choice epilogue at full CTA occupancy.
template <bool EPI>
__global__ void __launch_bounds__(32) k_rows_gather_warp(RowParams p) {
    extern __shared__ double wsm[]; // rowbuf[P64] + stage[32] 16-byte entries
    double* rowbuf = wsm;
    StageEntry* st = reinterpret_cast<StageEntry*>(wsm + p.P64);
    const int lane = threadIdx.x & 31;
    const int n = p.n;
    constexpr int AHEAD = ACO_GATHER_AHEAD;
    for (int i = p.row_begin + blockIdx.x; i < p.row_end; i += gridDim.x) {
        double* trow = p.tau + static_cast<size_t>(i) * p.P64;
        for (int j = lane; j < n; j += 32) rowbuf[j] = 0.0;
        __syncwarp();
        for (int g = 0; g < p.shards; ++g) {
            const int kbeg = g * p.S;
            const int cnt = min(p.S, p.m - kbeg);
            const int32_t* sc = p.succ + (static_cast<size_t>(g) * n + i) * p.S;
            const int32_t* pc = p.pred + (static_cast<size_t>(g) * n + i) * p.S;
            const double* wv = p.inv + static_cast<size_t>(g) * p.S;
            for (int k0 = 0; k0 < cnt; k0 += 16 * AHEAD) {
                int col[AHEAD];
                double w[AHEAD];
#pragma unroll
                for (int u = 0; u < AHEAD; ++u) {
                    const int k = k0 + 16 * u + (lane >> 1);
                    col[u] = -1;
                    w[u] = 0.0;
                    if (k < cnt) {
                        col[u] = __ldg((lane & 1) ? sc + k : pc + k);
                        w[u] = __ldg(wv + k);
                    }
                }
#pragma unroll
                for (int u = 0; u < AHEAD; ++u) {
                    // stage (column, weight) of the chunk as 16-byte entries;
                    // each lane folds the entries of its own column in lane
                    // (= ant) order — one LDS.128, one compare and one
                    // predicated DADD per entry — and every lane of a column
                    // stores the same folded value
                    const int cu = col[u];
                    st[lane] = StageEntry{cu, 0, w[u]};
                    __syncwarp();
                    double acc = cu >= 0 ? rowbuf[cu] : 0.0;
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const StageEntry e = st[q];
                        if (e.col == cu) acc = __dadd_rn(acc, e.w);
                    }
                    __syncwarp();
                    if (cu >= 0) rowbuf[cu] = acc;
                    __syncwarp();
                }
            }
        }
        if constexpr (!EPI) {
            double* drow = p.delta + static_cast<size_t>(i) * p.P64;
            for (int j = lane; j < n; j += 32) drow[j] = rowbuf[j];
            __syncwarp();
            continue;
        }
        double mx = 0.0;
        const int32_t* drow = p.dist + static_cast<size_t>(i) * p.P64;
        const double* erow = p.etab ? p.etab + static_cast<size_t>(i) * p.P64 : nullptr;
        // batches of EB columns per lane: all tau / dist loads, then all
        // eta^beta gathers, then the arithmetic (one warp per row has no other
        // latency hiding than these independent loads)
        constexpr int EB = 8;
        for (int j0 = 0; j0 < n; j0 += 32 * EB) {
            double tv[EB], eb[EB];
            int dv[EB];
#pragma unroll
            for (int u = 0; u < EB; ++u) {
                const int j = j0 + 32 * u + lane;
                tv[u] = j < n ? trow[j] : 0.0;
                dv[u] = (j < n && !erow) ? __ldg(drow + j) : 0;
            }
#pragma unroll
            for (int u = 0; u < EB; ++u) {
                const int j = j0 + 32 * u + lane;
                eb[u] = j < n ? (erow ? __ldg(erow + j) : __ldg(p.lut + dv[u])) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < EB; ++u) {
                const int j = j0 + 32 * u + lane;
                if (j < n) {
                    const double t = __dadd_rn(__dmul_rn(tv[u], p.keep), rowbuf[j]);
                    trow[j] = t;
                    const double c = (j == i) ? 0.0 : __dmul_rn(tau_pow(t, p.alpha, p.powtab), eb[u]);
                    p.choice64[static_cast<size_t>(i) * p.P64 + j] = c;
                    rowbuf[j] = c;
                    mx = fmax(mx, c);
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, off));
        __syncwarp();
        if (p.choice_nn) write_nn_row(p, rowbuf, i, lane);
        if (p.choice32) {
            const int sc = mx > 0.0 ? kScaleExp - ilogb(mx) : 0;
            if (lane == 0) p.scale_exp[i] = sc;
            write_stream_row<4>(p.choice32 + static_cast<size_t>(i) * p.PW, rowbuf, n, p.PW, p.C,
                                p.LA, sc, lane, 32, p.nat != 0);
        }
        if (p.choice_perm64) {
            write_stream_row<2>(p.choice_perm64 + static_cast<size_t>(i) * p.PW, rowbuf, n, p.PW,
                                p.C, p.LA, 0, lane, 32, p.nat != 0);
        }
        __syncwarp();
    }
}

// Device Philox self-test (aco_gpu_philox_uniform).
// ---------------------------------------------------------------------------
// Top-KT cache of every choice row for the nn selection's argmax fallback
// (select_next_nn, construction.hpp:108-120: argmax of w over the unvisited
// cities, the lowest index on ties).  Row i's list holds the KT best cities
// under the total order (w desc, index asc).  For any tabu set, the FIRST
// unvisited entry of the list is that argmax: every unvisited city outside
// the list is after every list entry in the order.  Only when all KT entries
// are visited does the construction scan the whole row.  A row whose
// candidate set overflows the scratch is marked invalid (entry 0 = -2) and
// always scans.  Rebuilt after every choice_info recomputation.
//
// Per row (one 256-thread CTA): 256 strided sub-range maxima straight from
// the row (8 loads in flight per thread); M = the KT-th largest of their
// high words (a 31-step bitwise search over block-wide counts), so at least
// KT cities have w >= M; a second pass over the row (L2-resident by then)
// collects those cities, which are ranked by the total order with integer
// compares of the bit patterns (w >= 0, so they order like w).  Bytes: 8 n^2 from HBM (+ the L2 re-read) + 4 KT n written.
#ifndef ACO_TOPK_K
#define ACO_TOPK_K 256 // entries per row of the argmax cache (128: 10k one GPU 1.5 ms slower construction, 0.3 ms faster rebuild)
#endif
constexpr int kTopK = ACO_TOPK_K;
constexpr int kTopThreads = 2 * kTopK; // one sub-range per thread
constexpr int kTopCap = kTopK <= 256 ? 6 * kTopK : 4 * kTopK; // static shared memory <= 48 KB
#ifndef ACO_TOPK_MINB
#define ACO_TOPK_MINB 8 // CTAs per SM the register budget must allow
#endif
#ifndef ACO_TOPK_REFINE
#define ACO_TOPK_REFINE 1 // second threshold over the candidates before ranking
#endif
#ifndef ACO_TOPK_B
#define ACO_TOPK_B 6 // row loads in flight per thread (8 spills at 32 registers)
#endif

// The K-th largest of the valid v (one per thread of an NT-thread block), 0
// when fewer than K are valid: 8-bit radix select, most significant digit
// first — per digit one shared histogram of the values still matching the
// prefix and one warp locating the digit where the count from the top
// reaches k (9 block barriers instead of a 31-step bitwise search).
// hist: 2 x 256 ints, sel: 2 ints of shared memory.
template <int NT>
__device__ __forceinline__ uint32_t block_kth_largest(uint32_t v, bool valid, int K, int* hist, int* sel) {
    const int tid = threadIdx.x;
    for (int b = tid; b < 256; b += NT) hist[b] = 0;
    if (__syncthreads_count(valid) < K) return 0u;
    uint32_t prefix = 0, mask = 0;
    int k = K;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        int* h = hist + (pass & 1) * 256;
        if (valid && (v & mask) == prefix) atomicAdd(&h[(v >> shift) & 255u], 1);
        __syncthreads();
        if (tid >= 32) { // the other buffer was last read in the previous pass
            int* h2 = hist + ((pass + 1) & 1) * 256;
            for (int b = tid - 32; b < 256; b += NT - 32) h2[b] = 0;
        } else {
            int c[8], sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = h[255 - 8 * tid - q]; // descending digits
                sum += c[q];
            }
            int incl = sum;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (tid >= off) incl += y;
            }
            const int excl = incl - sum;
            if (excl < k && k <= incl) {
                int acc = excl;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (acc < k && acc + c[q] >= k) {
                        sel[0] = 255 - 8 * tid - q;
                        sel[1] = k - acc;
                    }
                    acc += c[q];
                }
            }
        }
        __syncthreads();
        prefix |= static_cast<uint32_t>(sel[0]) << shift;
        mask |= 255u << shift;
        k = sel[1];
    }
    return prefix;
}

__global__ void __launch_bounds__(kTopThreads, ACO_TOPK_MINB * 256 / kTopThreads) k_row_topk(const double* __restrict__ choice, int n, int P64,
                                                  int32_t* __restrict__ topk) {
    // candidates as (bit pattern of w >= 0, which orders like w; index)
    __shared__ ulonglong2 cand[kTopCap];
    __shared__ int s_cnt;
    __shared__ int s_hist[512];
    __shared__ int s_sel[2];
    const int tid = threadIdx.x;
    constexpr int B = ACO_TOPK_B;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double* src = choice + static_cast<size_t>(i) * P64;
        if (tid == 0) s_cnt = 0;
        // sub-range q = j mod kTopThreads is thread q's: its maximum straight from HBM
        double m0 = -1.0;
        for (int k0 = 0; k0 < n; k0 += kTopThreads * B) {
            double v[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int j = k0 + kTopThreads * u + tid;
                v[u] = j < n ? __ldg(src + j) : -1.0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u) m0 = fmax(m0, v[u]);
        }
        // M: the largest high word H (sign, exponent, 20 mantissa bits) such
        // that >= KT sub-range maxima have high word >= H, found bit by bit
        // with block-wide counts; M = H:0 is <= each of those maxima, so at
        // least KT cities have w >= M.  (Fewer than KT non-empty sub-ranges,
        // i.e. n < KT: M = 0 and every city is a candidate.)
        const bool valid = m0 >= 0.0;
        const uint32_t hi = valid ? static_cast<uint32_t>(__double_as_longlong(m0) >> 32) : 0u;
        // (the K-th largest high word is exactly that H)
        const uint32_t H = block_kth_largest<kTopThreads>(hi, valid, kTopK, s_hist, s_sel);
        const double M = __longlong_as_double(static_cast<long long>(H) << 32);
        // second pass over the (now L2-resident) row: collect w >= M
        for (int k0 = 0; k0 < n; k0 += kTopThreads * B) {
            double v[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int j = k0 + kTopThreads * u + tid;
                v[u] = j < n ? __ldg(src + j) : -1.0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                if (v[u] >= M) {
                    const int pos = atomicAdd(&s_cnt, 1);
                    if (pos < kTopCap)
                        cand[pos] = make_ulonglong2(static_cast<unsigned long long>(__double_as_longlong(v[u])),
                                                    static_cast<unsigned long long>(k0 + kTopThreads * u + tid));
                }
            }
        }
        __syncthreads();
        int c = s_cnt;
        int32_t* out = topk + static_cast<size_t>(i) * kTopK;
        if (c > kTopCap) {
            if (tid == 0) out[0] = -2; // invalid: the construction scans the row
        } else {
#if ACO_TOPK_REFINE
            if (c > kTopK + 16 && c <= kTopThreads) {
                // second threshold, over the candidates' own high words: a
                // candidate below H2 is below every candidate at or above
                // it, and >= KT are at or above, so only those are ranked
                const bool own = tid < c;
                const ulonglong2 e = own ? cand[tid] : make_ulonglong2(0ull, 0ull);
                const uint32_t h = static_cast<uint32_t>(e.x >> 32);
                const uint32_t H2 = block_kth_largest<kTopThreads>(h, own, kTopK, s_hist, s_sel);
                if (tid == 0) s_cnt = 0;
                __syncthreads();
                if (own && h >= H2) cand[atomicAdd(&s_cnt, 1)] = e;
                __syncthreads();
                c = s_cnt;
            }
#endif
            // rank under (w desc, index asc), branch-free integer compares
            for (int a = tid; a < c; a += kTopThreads) {
                const ulonglong2 ea = cand[a];
                int r = 0;
                for (int b = 0; b < c; ++b) {
                    const ulonglong2 eb = cand[b];
                    r += static_cast<int>((eb.x > ea.x) | ((eb.x == ea.x) & (eb.y < ea.y)));
                }
                if (r < kTopK) out[r] = static_cast<int32_t>(ea.y);
            }
            for (int r = c + tid; r < kTopK; r += kTopThreads) out[r] = -1; // n < KT: end of list
        }
        __syncthreads();
    }
}

__global__ void k_philox_test(uint64_t seed, uint32_t it, uint32_t ant, int count,
                              const uint32_t* steps, const uint32_t* draws, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = philox_uniform(seed, it, ant, steps[i], draws[i]);
}

// Unit harness for libm_pow (aco_gpu_libm_pow, the creation self-test).
__global__ void k_libm_pow(const double* __restrict__ xs, const double* __restrict__ ys, int count,
                           const LibmPowTables* __restrict__ T, double* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        out[i] = libm_pow(xs[i], ys[i], T);
}

} // namespace acob200
