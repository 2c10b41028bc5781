// Two ants per warp: the roulette construction kernel for n <= 2560 with the
// fp32 stream (the pr2392 hot path).
//
// Same algorithm and the same three certification tiers as
// k_construct_roulette (construct.cuh), but lanes 0-15 run ant 2p and lanes
// 16-31 ant 2p+1, each lane owning C = 4*NV contiguous cities of its ant's
// row (rows are streamed in the LA = 16 lane-major layout: a line holds 16
// lanes' 16-byte vectors + 1 pad slot).  Pass 1 costs the same per ant, but
// every step's scans, search, certification, TMA/tabu bookkeeping and loop
// control are issued once per warp for TWO ants, and register pressure
// disappears (8-9 warps per SM instead of 16-17).  All warp collectives are
// either half-segmented (width 16) or ballots split per half.
#pragma once

#include "construct.cuh"

namespace acob200 {

__device__ __forceinline__ unsigned half_of(unsigned b, int hb) { return (b >> hb) & 0xFFFFu; }

// lowest unvisited city of one half's ant (construction.hpp:31-35)
__device__ __forceinline__ int lowest_unvisited_half(const uint32_t* tabu, int words, int hl,
                                                     int hb) {
    for (int w0 = 0; w0 < words; w0 += 16) {
        const int wd = w0 + hl;
        const uint32_t fr = wd < words ? ~tabu[wd] : 0u;
        const unsigned b = half_of(__ballot_sync(kFull, fr != 0u), hb);
        if (b) {
            const int src = __ffs(b) - 1;
            const uint32_t fb = __shfl_sync(kFull, fr, hb + src);
            return (w0 + src) * 32 + __ffs(fb) - 1;
        }
    }
    return -1;
}

// Tier 2 for both halves at once: fp64 prefix sums over the fp32 row in the
// half's shared buffer (quantisation-only error).  Returns the certified city
// of this lane's half, or -1.  Read-only on shared memory.
template <int NV>
__device__ __noinline__ int certify_fp64_pair(const float* buf, const uint32_t* tabu, int n,
                                              double u, int hl, int hb) {
    constexpr int C = 4 * NV, LP = 17, NWIN = C / 32;
    const double e_rel = (2.0 * 0x1.0p-24 + (double)(C + 32) * 0x1.0p-53 +
                          (double)(n + 8) * 0x1.0p-53) * (1.0 + 0x1.0p-16);
    const double abs_q = (double)n * 0x1.0p-149;
    uint32_t win[NWIN];
#pragma unroll
    for (int i = 0; i < NWIN; ++i) win[i] = tabu[(hl * C >> 5) + i];
    const float4* rv = reinterpret_cast<const float4*>(buf) + hl;
    double acc = 0.0;
#pragma unroll 4
    for (int t = 0; t < NV; ++t) {
        const float4 v = rv[t * LP];
        const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = 4 * t + q;
            if (!((win[e >> 5] >> (e & 31)) & 1u)) acc += static_cast<double>(xs[q]);
        }
    }
    double d = acc;
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
        const double y = __shfl_up_sync(kFull, d, off, 16);
        if (hl >= off) d += y;
    }
    const double T = __shfl_sync(kFull, d, hb + 15);
    const bool good = (T > 0.0) && (T < 1e300);
    const double t = u * T;
    const unsigned lb = half_of(__ballot_sync(kFull, good && d > t), hb);
    const int L = lb ? __ffs(lb) - 1 : -1;
    int J = -1;
    bool cert = false;
    if (hl == L) {
        double a = d - acc; // exclusive prefix of this lane
        for (int e = 0; e < C; ++e) {
            if ((win[e >> 5] >> (e & 31)) & 1u) continue;
            const int tv = e >> 2, q = e & 3;
            const double x = static_cast<double>(buf[(tv * LP + hl) * 4 + q]);
            const double na = a + x;
            if (x > 0.0 && na > t) {
                const double Thi = T * (1.0 + 0x1.0p-16) + abs_q;
                const double Mt = (e_rel + 0x1.0p-50) * (u * Thi) + abs_q;
                cert = (na * (1.0 - e_rel) - 2.0 * abs_q > t + Mt) &&
                       (a + e_rel * na + 2.0 * abs_q < t - Mt);
                J = hl * C + e;
                break;
            }
            a = na;
        }
    }
    const int srcl = hb + (L >= 0 ? L : 0);
    J = __shfl_sync(kFull, J, srcl);
    const bool c2 = __shfl_sync(kFull, cert, srcl);
    return (L >= 0 && c2 && J >= 0 && J < n) ? J : -1;
}

// Tier 3 for the halves with `active` set (both halves execute the warp
// collectives): exact replay of select_next_roulette over the fp64 row,
// staged through the half's buffer with TMA; every lane of the half folds
// every weight in ascending order (construction.hpp:42-68).
__device__ __noinline__ int exact_walk_pair(const double* __restrict__ row, const uint32_t* tabu,
                                            int n, int words, double u, int hl, int hb,
                                            bool active, double* chunk_start, double* stage,
                                            uint32_t stage_bytes, uint64_t* bar,
                                            uint32_t& phase) {
    const int nch = (n + 31) >> 5;
    const int piece = static_cast<int>(stage_bytes / 256) * 32;
    double acc = 0.0;
    int last_positive = -1;
    for (int p0 = 0; p0 < n; p0 += piece) {
        const int cnt = min(piece, n - p0);
        const uint32_t bytes = static_cast<uint32_t>(((cnt * 8) + 15) & ~15);
        __syncwarp();
        if (active && hl == 0) {
            fence_proxy_async_smem();
            mbar_expect_tx(bar, bytes);
            tma_row(stage, row + p0, bytes, bar);
        }
        __syncwarp();
        if (active) {
            mbar_wait(bar, phase);
            phase ^= 1u;
        }
        for (int c = p0 >> 5; c < ((p0 + cnt + 31) >> 5); ++c) {
            const int base = c << 5;
            const uint32_t vis = tabu[c];
            const double2* s2 = reinterpret_cast<const double2*>(stage + (base - p0));
            if (hl == 0) chunk_start[c] = acc;
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
    // every lane of both halves runs the same collectives below (no early
    // returns: the halves may be in different branches of the reference)
    const bool zero = !(acc > 0.0);
    const int lowest = lowest_unvisited_half(tabu, words, hl, hb);
    const double target = u * acc;
    int ch = -1;
    for (int c0 = 0; c0 < nch; c0 += 16) {
        const int c = c0 + hl;
        const double end = c < nch ? (c + 1 < nch ? chunk_start[c + 1] : acc) : -1.0;
        const unsigned b = half_of(__ballot_sync(kFull, c < nch && end > target), hb);
        if (ch < 0 && b) ch = c0 + __ffs(b) - 1;
    }
    const int base = (ch >= 0 ? ch : 0) << 5;
    const int j0 = base + hl, j1 = base + 16 + hl;
    const double w0 = (j0 < n && !tabu_test(tabu, j0)) ? __ldg(row + j0) : 0.0;
    const double w1 = (j1 < n && !tabu_test(tabu, j1)) ? __ldg(row + j1) : 0.0;
    double a2 = chunk_start[ch >= 0 ? ch : 0], m0 = 0.0, m1 = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        a2 += __shfl_sync(kFull, w0, hb + q);
        m0 = (q == hl) ? a2 : m0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        a2 += __shfl_sync(kFull, w1, hb + q);
        m1 = (q == hl) ? a2 : m1;
    }
    const unsigned c0b = half_of(__ballot_sync(kFull, m0 > target), hb);
    const unsigned c1b = half_of(__ballot_sync(kFull, m1 > target), hb);
    if (zero) return lowest;                                             // :52
    if (ch < 0) return last_positive >= 0 ? last_positive : lowest;      // :66
    return c0b ? base + __ffs(c0b) - 1 : base + 16 + __ffs(c1b) - 1;     // first prefix > target
}

template <int NV>
__global__ void __maxnreg__(168) k_construct_roulette_pair(ConstructParams p) {
    constexpr int C = 4 * NV;           // cities per lane
    constexpr int LP = 17;              // vector slots per line (16 lanes + pad)
    constexpr int NWIN = C / 32;
    constexpr int GV = 4, NG = (NV + GV - 1) / GV, GE = 16;
    constexpr int D1 = 4 + ceil_log2<NG>();
    static_assert(NV % 8 == 0, "chunks must be word aligned");

    const int lane = threadIdx.x & 31, hl = lane & 15, hb = lane & 16, h = lane >> 4;
    const int n = p.n;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* hbase = smem_raw + static_cast<size_t>(h) * p.half_smem;
    uint64_t* bar = reinterpret_cast<uint64_t*>(hbase);
    float* buf = reinterpret_cast<float*>(hbase + 128);
    uint32_t* tabu = reinterpret_cast<uint32_t*>(hbase + 128 + static_cast<size_t>(p.PW) * 4);
    double* chunk_start = reinterpret_cast<double*>(tabu + p.tabu_words);
    float* gx = reinterpret_cast<float*>(chunk_start + ((n + 31) >> 5));
    const float* __restrict__ wbase = static_cast<const float*>(p.w);
    const uint32_t row_bytes = static_cast<uint32_t>(p.PW * 4);

    // bound: fp32 quantisation (x2) + fp32 adds on any prefix path (tree D1,
    // lane scan 4, group scan 4, city scan 4, 3 more) + fp64 + reference gamma_n
    const double e_rel = ((double)(2 + D1 + 4 + 4 + 4 + 3) * 0x1.0p-24 +
                          (double)(n + 16) * 0x1.0p-53) * (1.0 + 0x1.0p-16);
    const double abs_q = (double)n * 0x1.0p-149;
    const double lo_f = 1.0 - e_rel;

    if (hl == 0) mbar_init(bar, 1);
    __syncwarp();
    uint32_t phase = 0;

    const int pairs = (p.mloc + 1) >> 1;
    for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
        const int kl_raw = 2 * pr + h;
        const bool live = kl_raw < p.mloc;          // the odd tail duplicates ant 2pr
        const int kl = live ? kl_raw : 2 * pr;
        const uint32_t kg = static_cast<uint32_t>(p.ant_begin + kl);
        int32_t* tour = p.tours + static_cast<size_t>(kl) * (n + 1);
        for (int wd = hl; wd < p.tabu_words; wd += 16) {
            const int c0 = wd * 32;
            tabu[wd] = (c0 + 32 <= n) ? 0u : (c0 >= n ? kFull : (kFull << (n - c0)));
        }
        const int start = start_city(p, kg);
        __syncwarp();
        if (hl == 0) {
            tabu[start >> 5] |= 1u << (start & 31);
            if (live) tour[0] = start;
        }
        int cur = start;
        unsigned long long fb = 0;
        bool prefetched = false;
        double ubatch = 0.0;

        for (int step = 1; step < n; ++step) {
            if (!prefetched && hl == 0) {
                fence_proxy_async_smem();
                mbar_expect_tx(bar, row_bytes);
                tma_row(buf, wbase + static_cast<size_t>(cur) * p.PW, row_bytes, bar);
            }
            // draw 0 of steps step..step+15: lane hl of a half holds step + hl
            if (((step - 1) & 15) == 0)
                ubatch = philox_uniform(p.seed, p.iteration, kg, static_cast<uint32_t>(step + hl), 0);
            const double u = __shfl_sync(kFull, ubatch, hb + ((step - 1) & 15));
            __syncwarp();
            mbar_wait(bar, phase);
            phase ^= 1u;
            prefetched = false;

            // ---- pass 1: masked lane sums (group sums kept for the search)
            uint32_t win[NWIN];
#pragma unroll
            for (int i = 0; i < NWIN; ++i) win[i] = tabu[(hl * C >> 5) + i];
            const float4* rv = reinterpret_cast<const float4*>(buf) + hl;
            float gs[NG];
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                float x[GE];
#pragma unroll
                for (int tt = 0; tt < GV; ++tt) {
                    const int tv = g * GV + tt;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (tv < NV) v = rv[tv * LP];
                    x[tt * 4 + 0] = v.x; x[tt * 4 + 1] = v.y; x[tt * 4 + 2] = v.z; x[tt * 4 + 3] = v.w;
                }
#pragma unroll
                for (int e = 0; e < GE; ++e) {
                    const int ee = g * GE + e;
                    if (ee < C && ((win[ee >> 5] >> (ee & 31)) & 1u)) x[e] = 0.f;
                }
                gs[g] = tree_sum_packed<GE>(x);
            }
            float gsc[NG]; // group sums survive the (in-place) lane tree
#pragma unroll
            for (int g = 0; g < NG; ++g) gsc[g] = gs[g];
            float d = tree_sum<float, NG>(gs);
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) {
                const float y = __shfl_up_sync(kFull, d, off, 16);
                if (hl >= off) d += y;
            }
            const float T = __shfl_sync(kFull, d, hb + 15);
            const double Td = static_cast<double>(T);
            const double tdd = u * Td;
            const float t = static_cast<float>(tdd);
            const double Thi = Td * (1.0 + 0x1.0p-16) + abs_q;
            const double Mt = (e_rel + 4.0 * 0x1.0p-24) * (u * Thi) + abs_q;
            const double A = tdd + Mt + 2.0 * abs_q;
            const double B = tdd - Mt - 2.0 * abs_q;
            const bool good = (T > 0.f) && (Td < 1e300);

            // ---- crossing lane L of each half, then its group, then its city
            const unsigned lb = half_of(__ballot_sync(kFull, good && d > t), hb);
            const int L = lb ? __ffs(lb) - 1 : -1;
            const float myprev = __shfl_sync(kFull, d, hb + (L > 0 ? L - 1 : 0));
            const float exclL = L > 0 ? myprev : 0.f;
            if (hl == L) {
#pragma unroll
                for (int g = 0; g < NG; ++g) gx[g] = gsc[g];
            }
            __syncwarp();
            const float gv = (L >= 0 && hl < NG) ? gx[hl] : 0.f;
            float gi = gv;
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) {
                const float y = __shfl_up_sync(kFull, gi, off, 16);
                if (hl >= off) gi += y;
            }
            const unsigned gb = half_of(__ballot_sync(kFull, L >= 0 && hl < NG && exclL + gi > t), hb);
            const int G = gb ? __ffs(gb) - 1 : -1;
            const float gprev = __shfl_sync(kFull, gi, hb + (G > 0 ? G - 1 : 0));
            const float gbefore = exclL + (G > 0 ? gprev : 0.f);
            float xv = 0.f;
            const int e = (G >= 0 ? G : 0) * GE + hl; // city offset in lane L's chunk
            const int city = (L >= 0 ? L : 0) * C + e;
            if (G >= 0 && e < C) {
                xv = buf[((e >> 2) * LP + L) * 4 + (e & 3)];
                if (tabu_test(tabu, city)) xv = 0.f;
            }
            float xi = xv;
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) {
                const float y = __shfl_up_sync(kFull, xi, off, 16);
                if (hl >= off) xi += y;
            }
            const float xe = __shfl_up_sync(kFull, xi, 1, 16);
            const unsigned eb = half_of(__ballot_sync(kFull, G >= 0 && xv > 0.f && gbefore + xi > t), hb);
            const int E = eb ? __ffs(eb) - 1 : -1;
            bool cert = false;
            if (hl == E) {
                const double Pj = static_cast<double>(gbefore + xi);
                const double Pprev = static_cast<double>(gbefore + (hl > 0 ? xe : 0.f));
                cert = (Pj * lo_f > A) && (Pprev + e_rel * Pj < B) && city < n;
                if (cert && step + 1 < n) { // speculative refill of this half's buffer
                    mbar_expect_tx(bar, row_bytes);
                    tma_row(buf, wbase + static_cast<size_t>(city) * p.PW, row_bytes, bar);
                }
            }
            const unsigned cb = half_of(__ballot_sync(kFull, cert), hb);
            bool ok = cb != 0u;
            int next = __shfl_sync(kFull, city, hb + (cb ? __ffs(cb) - 1 : 0));
            prefetched = ok && step + 1 < n;

            // ---- tiers 2 and 3 (rare), per half
            if (__ballot_sync(kFull, !ok)) {
                const int j2 = certify_fp64_pair<NV>(buf, tabu, n, u, hl, hb);
                if (!ok && j2 >= 0) {
                    ok = true;
                    next = j2;
                }
                if (__ballot_sync(kFull, !ok)) {
                    const int j3 = exact_walk_pair(p.w64 + static_cast<size_t>(cur) * p.P64, tabu, n,
                                                   p.tabu_words, u, hl, hb, !ok, chunk_start,
                                                   reinterpret_cast<double*>(buf),
                                                   row_bytes & ~255u, bar, phase);
                    if (!ok) {
                        next = j3;
                        ++fb;
                    }
                }
            }
            if (hl == 0) {
                tabu[next >> 5] |= 1u << (next & 31);
                if (live) tour[step] = next;
            }
            cur = next;
        }
        if (hl == 0) {
            if (live) tour[n] = start;
            if (live && fb) atomicAdd(p.fallbacks, fb);
        }
        __syncwarp();
    }
}

} // namespace acob200
