// Team roulette construction: K warps (one CTA) per ant, for colonies too
// small to fill the GPU with one warp per ant (pr1002 on one B200: 6.8 ants
// per SM; pr2392 sharded over 2/4/8 GPUs: 8.1/4.0/2.0 ants per SM).  With
// one warp per ant such a colony is bound by the per-step dependent chain
// (~1850 cycles per step at one ant per SM), not by L2; K warps
// split every step's row so each warp's chain (chunk sums, lane scan) is K
// times shorter.
//
// Same selection rule, certification and fallbacks as k_construct_roulette
// (construct.cuh; select_next_roulette, construction.hpp:42-68), bit-exact by
// the same argument.  The streamed fp32 row uses the multi-round layout of
// stream_pos with R = K rounds of 32 lanes x C cities: warp w owns round w.
// Per step:
//   1. every warp waits for the row (one TMA bulk copy, mbarrier `bar`),
//      tree-sums its lanes' masked chunks and scans them (fp32);
//   2. the K warp totals meet in shared memory (one __syncthreads);
//   3. every warp folds the K totals in warp order (the same adds in every
//      warp, so all agree on T, t = u*T and the crossing warp W);
//   4. warp W alone runs the group walk and certification over its round
//      (base = the exclusive sum of warps < W); its certifying lane marks the
//      tabu, writes the tour and issues the next row's TMA.  If nothing
//      certifies, warp W runs the fp64 tiers (certify_fp64 over all K rounds,
//      then exact_walk with its own staging mbarrier) and issues the TMA.
// The other warps go straight to step 1 of the next step: the mbarrier
// completion of the next row orders the tabu update before their reads
// (the issuing thread's arrive has release semantics, try_wait acquire).
#pragma once

#include "construct.cuh"

namespace acob200 {

template <int K, int NV>
__global__ void __launch_bounds__(32 * K) k_construct_team(ConstructParams p) {
    using AT = float;
    constexpr int V = 4;
    constexpr int C = NV * V;
    constexpr int NWIN = (C + 31) / 32;
    constexpr int GV = 4;
    constexpr int NG = (NV + GV - 1) / GV;
    constexpr int GE = GV * V;
    constexpr int D1 = ceil_log2<GE>() + ceil_log2<NG>();
    static_assert(K >= 2 && K <= 8, "2..8 warps per ant");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);          // row barrier
    uint64_t* bar_fb = bar + 1;                                      // [K] staging barriers
    float* tot = reinterpret_cast<float*>(smem_raw + 80);            // [2][8] warp totals
    int* cur_slot = reinterpret_cast<int*>(smem_raw + 144);          // [2] current city by step parity
    float* buf = reinterpret_cast<float*>(smem_raw + 256);
    uint32_t* tabu = reinterpret_cast<uint32_t*>(smem_raw + 256 + static_cast<size_t>(p.PW) * 4);
    double* chunk_start = reinterpret_cast<double*>(tabu + p.tabu_words);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = p.n;
    const float* __restrict__ wbase = static_cast<const float*>(p.w);
    const uint32_t row_bytes = static_cast<uint32_t>(p.PW * 4);

    // Error bound as in k_construct_roulette with MAXR = K (round bases) plus
    // the base add of the crossing warp and 2 more of slack.
    constexpr double ulp_at = 0x1.0p-24;
    const double e_rel = ((double)(D1 + 5 + K + 1 + 2 + 5 + 4 + 3 + 3) * ulp_at + 2.0 * 0x1.0p-24 +
                          (double)(n + 8) * 0x1.0p-53) * (1.0 + 0x1.0p-16);
    const double abs_q = (double)n * 0x1.0p-149;
    const double lo_f = 1.0 - e_rel;

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        for (int w = 0; w < K; ++w) mbar_init(bar_fb + w, 1);
    }
    __syncthreads();
    uint32_t phase = 0, phase_fb = 0;

    for (int kl = blockIdx.x; kl < p.mloc; kl += gridDim.x) {
        const uint32_t kg = static_cast<uint32_t>(p.ant_begin + kl);
        int32_t* tour = p.tours + static_cast<size_t>(kl) * (n + 1);
        for (int wd = threadIdx.x; wd < p.tabu_words; wd += 32 * K) {
            const int c0 = wd * 32;
            tabu[wd] = c0 + 32 <= n ? 0u : (c0 >= n ? kFull : (kFull << (n - c0)));
        }
        const int start = start_city(p, kg);
        __syncthreads();
        if (threadIdx.x == 0) {
            tabu[start >> 5] |= 1u << (start & 31);
            tour[0] = start;
            cur_slot[0] = start;
            fence_proxy_async_smem();
            mbar_expect_tx(bar, row_bytes);
            tma_row(buf, wbase + static_cast<size_t>(start) * p.PW, row_bytes, bar);
        }
        unsigned long long fb = 0;
        double ubatch = 0.0;

        for (int step = 1; step < n; ++step) {
            if (((step - 1) & 31) == 0)
                ubatch = philox_uniform(p.seed, p.iteration, kg, static_cast<uint32_t>(step + lane), 0);
            const double u = __shfl_sync(kFull, ubatch, (step - 1) & 31);
            mbar_wait(bar, phase);
            phase ^= 1u;

            // 1. this warp's round: masked chunk sums, lane-local group prefixes
            const int cbase = warp * 32 * C + lane * C;
            uint32_t win[NWIN];
            {
                const int w0 = cbase >> 5, sh = cbase & 31;
#pragma unroll
                for (int i = 0; i < NWIN; ++i) win[i] = __funnelshift_r(tabu[w0 + i], tabu[w0 + i + 1], sh);
            }
            const float4* rv = reinterpret_cast<const float4*>(buf + warp * kLP * C) + lane;
            float gs[NG], gsr[NG];
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                float x[GE];
#pragma unroll
                for (int tt = 0; tt < GV; ++tt) {
                    const int tv = g * GV + tt;
                    const float4 v = tv < NV ? rv[tv * kLP] : make_float4(0.f, 0.f, 0.f, 0.f);
                    x[tt * 4 + 0] = v.x; x[tt * 4 + 1] = v.y; x[tt * 4 + 2] = v.z; x[tt * 4 + 3] = v.w;
                }
#pragma unroll
                for (int e = 0; e < GE; ++e) {
                    const int ee = g * GE + e;
                    if (ee < C && ((win[ee >> 5] >> (ee & 31)) & 1u)) x[e] = 0.f;
                }
                gs[g] = tree_sum_packed<GE>(x);
            }
            gsr[0] = gs[0];
#pragma unroll
            for (int g = 1; g < NG; ++g) gsr[g] = gsr[g - 1] + gs[g];
            const float incl = warp_inclusive_scan(tree_sum<float, NG>(gs));
            const int par = (step & 1) * 8;
            if (lane == 31) tot[par + warp] = incl;
            __syncthreads();

            // 3. fold the K warp totals in warp order (identical in every warp)
            AT cum[K];
            cum[0] = tot[par];
#pragma unroll
            for (int v = 1; v < K; ++v) cum[v] = cum[v - 1] + tot[par + v];
            const AT T = cum[K - 1];
            const double Td = static_cast<double>(T);
            const double tdd = u * Td;
            const AT t = static_cast<AT>(tdd);
            int W = -1;
            const bool tot_ok = (T > AT(0)) && (Td < 1e300);
            if (tot_ok) {
#pragma unroll
                for (int v = K - 1; v >= 0; --v) W = cum[v] > t ? v : W;
            }
            const int resolver = W >= 0 ? W : 0;
            if (warp != resolver) continue; // next row arrives through `bar`

            // 4. crossing warp: group walk + certification over its round
            int next = -1;
            bool ok = false;
            if (W >= 0) {
                const double Thi = Td * (1.0 + 0x1.0p-16) + abs_q;
                const double Mt = (e_rel + 4.0 * ulp_at) * (u * Thi) + abs_q;
                const double A = tdd + Mt + 2.0 * abs_q;
                const double B = tdd - Mt - 2.0 * abs_q;
                AT baseW = AT(0); // cum[W - 1], selected without a local-memory index
#pragma unroll
                for (int v = 0; v + 1 < K; ++v) baseW = (v + 1 == W) ? cum[v] : baseW;
                const AT exo = __shfl_up_sync(kFull, incl, 1);
                const AT excl_own = baseW + (lane == 0 ? AT(0) : exo);
                const unsigned lb = __ballot_sync(kFull, baseW + incl > t);
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
                int J = -1;
                bool cert = false;
                if (lb) {
                    const int L = __ffs(lb) - 1;
                    const int G = __shfl_sync(kFull, Gown, L);
                    const AT baseG = __shfl_sync(kFull, bG, L);
                    if (G < NG) {
                        const int k = lane & 3;
                        const int tv = G * GV + k;
                        const int c0 = W * 32 * C + L * C + tv * 4;
                        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                        uint32_t bits4 = 0xFu;
                        if (tv < NV) {
                            v = reinterpret_cast<const float4*>(buf + W * kLP * C)[tv * kLP + L];
                            bits4 = __funnelshift_r(tabu[c0 >> 5], tabu[(c0 >> 5) + 1], c0 & 31);
                        }
                        const AT x0 = (bits4 & 1u) ? AT(0) : v.x;
                        const AT x1 = (bits4 & 2u) ? AT(0) : v.y;
                        const AT x2 = (bits4 & 4u) ? AT(0) : v.z;
                        const AT x3 = (bits4 & 8u) ? AT(0) : v.w;
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
                        if (x3 > AT(0) && p3 > t) { E = 3; Pj32 = p3; Pp32 = p2; }
                        if (x2 > AT(0) && p2 > t) { E = 2; Pj32 = p2; Pp32 = p1; }
                        if (x1 > AT(0) && p1 > t) { E = 1; Pj32 = p1; Pp32 = p0; }
                        if (x0 > AT(0) && p0 > t) { E = 0; Pj32 = p0; Pp32 = kb; }
                        const unsigned qb = __ballot_sync(kFull, lane < 4 && E >= 0);
                        const bool mine = qb != 0u && lane == __ffs(qb) - 1;
                        const double Pj = static_cast<double>(Pj32);
                        const double Pprev = static_cast<double>(Pp32);
                        const int Jc = c0 + E;
                        J = mine ? Jc : -1;
                        cert = mine && (Pj * lo_f > A) && (Pprev + e_rel * Pj < B) && Jc < n;
                    }
                }
                if (cert) { // every read of buf and tabu this step has returned
                    tabu[J >> 5] |= 1u << (J & 31);
                    tour[step] = J;
                    if (step + 1 < n) {
                        mbar_expect_tx(bar, row_bytes);
                        tma_row(buf, wbase + static_cast<size_t>(J) * p.PW, row_bytes, bar);
                    }
                }
                const unsigned cb = __ballot_sync(kFull, cert);
                ok = cb != 0u;
                if (ok) next = __shfl_sync(kFull, J, __ffs(cb) - 1);
            }
            if (!ok) {
                // fp64 tiers over the whole row (all K rounds), this warp alone;
                // the other warps are parked on `bar` and read nothing.
                const int cur_w = cur_slot[(step - 1) & 1]; // published by step-1's resolver
                next = certify_fp64<float, NV, K>(buf, tabu, n, K, u, lane);
                if (next < 0) {
                    next = exact_walk(p.w64 + static_cast<size_t>(cur_w) * p.P64, tabu, n,
                                      p.tabu_words, u, lane, chunk_start,
                                      reinterpret_cast<double*>(buf), row_bytes & ~255u,
                                      bar_fb + warp, phase_fb);
                    phase_fb ^= static_cast<uint32_t>(exact_walk_pieces(n, row_bytes & ~255u) & 1);
                    ++fb;
                }
                __syncwarp();
                if (lane == 0) {
                    tabu[next >> 5] |= 1u << (next & 31);
                    tour[step] = next;
                    if (step + 1 < n) {
                        fence_proxy_async_smem();
                        mbar_expect_tx(bar, row_bytes);
                        tma_row(buf, wbase + static_cast<size_t>(next) * p.PW, row_bytes, bar);
                    }
                }
            }
            // publish the current city for whichever warp resolves the next
            // step (read after that step's __syncthreads)
            if (lane == 0) cur_slot[step & 1] = next;
        }
        __syncthreads();
        if (threadIdx.x == 0) tour[n] = start;
        if (lane == 0 && fb) atomicAdd(p.fallbacks, fb);
    }
}

} // namespace acob200
