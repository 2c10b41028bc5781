// libaco_probe.so — measurement helpers for the roofline denominators
// (not on the product path).  SURVEY §8(d): "measure the L2 bandwidth with a
// read kernel over a resident buffer of ~50% of the L2, 16-byte loads on all
// SMs"; the same kernel over a buffer far larger than L2 gives HBM read BW.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {

template <int CG>
__global__ void k_read(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) {
        // CG = 1: ld.global.cg (cached in L2 only), so no repetition can hit in L1
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
             i += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const float4 v = CG ? __ldcg(p + i) : __ldg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1234.5f) *sink = acc; // never true for a zero buffer; keeps the loads
}

} // namespace

extern "C" int aco_probe_read_bw_mode(int device, size_t bytes, int reps, int iters, int cg,
                                      double* gbps, double* ms_out) {
    auto kern = cg ? k_read<1> : k_read<0>;
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    float4* buf = nullptr;
    float* sink = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 2;
    cudaMalloc(&sink, sizeof(float));
    cudaMemset(buf, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const size_t n4 = bytes / 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<sms * 8, 512>>>(buf, n4, 1, sink); // warm (L2-resident when it fits)
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int it = 0; it < iters; ++it) {
        cudaEventRecord(a);
        kern<<<sms * 8, 512>>>(buf, n4, reps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    *ms_out = best;
    *gbps = static_cast<double>(bytes) * reps / (best * 1e-3) / 1e9;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// red.global.add.f64 throughput at pseudo-random addresses over a buffer of
// `bytes` (the deposit's access pattern: no locality, no contention) — the
// atomic roofline of k_deposit_atomic (46 MB: L2-resident like pr2392's tau;
// 800 MB: HBM-backed like 10k's).
__global__ void k_red(double* __restrict__ buf, size_t ncells, size_t nops, unsigned seed) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nops;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        unsigned long long h = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        atomicAdd(buf + (h % ncells), 1e-9);
    }
}

extern "C" int aco_probe_red(int device, size_t bytes, size_t nops, int iters, double* gops,
                             double* ms_out) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    double* buf = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 2;
    cudaMemset(buf, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const size_t ncells = bytes / sizeof(double);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_red<<<sms * 8, 256>>>(buf, ncells, nops, 1u);
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int it = 0; it < iters; ++it) {
        cudaEventRecord(a);
        k_red<<<sms * 8, 256>>>(buf, ncells, nops, 7u + it);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    *ms_out = best;
    *gops = static_cast<double>(nops) / (best * 1e-3) / 1e9;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

extern "C" int aco_probe_read_bw(int device, size_t bytes, int reps, int iters, double* gbps,
                                 double* ms_out) {
    return aco_probe_read_bw_mode(device, bytes, reps, iters, 0, gbps, ms_out);
}

// ---- dependent-chain latency probes (cycles per op, one warp) -------------
namespace {
template <int OP>
__global__ void k_chain(double* out, float* outf, int iters, long long* cyc, double seed) {
    double d = seed, e = seed * 0.5;
    float f = static_cast<float>(seed), g = static_cast<float>(seed) * 0.5f;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (OP == 0) d = __dadd_rn(d, e);
            if (OP == 1) d = __dmul_rn(d, e);
            if (OP == 2) d = __fma_rn(d, e, e);
            if (OP == 3) f = __fadd_rn(f, g);
            if (OP == 4) d = static_cast<double>(static_cast<float>(d) + g);
            if (OP == 5) d = __shfl_sync(0xffffffffu, d, (threadIdx.x + 1) & 31) + e;
            if (OP == 6) f = __shfl_sync(0xffffffffu, f, (threadIdx.x + 1) & 31);
            if (OP == 7) { d = (d > e) ? d - e : d + e; }
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    out[threadIdx.x] = d;
    outf[threadIdx.x] = f;
}
} // namespace

extern "C" int aco_probe_latency(int device, int op, int iters, double* cycles_per_op) {
    cudaSetDevice(device);
    double* out; float* outf; long long* cyc;
    cudaMalloc(&out, 32 * sizeof(double)); cudaMalloc(&outf, 32 * sizeof(float));
    cudaMalloc(&cyc, sizeof(long long));
    void (*fns[])(double*, float*, int, long long*, double) = {k_chain<0>, k_chain<1>, k_chain<2>, k_chain<3>,
                                                              k_chain<4>, k_chain<5>, k_chain<6>, k_chain<7>};
    fns[op]<<<1, 32>>>(out, outf, iters, cyc, 1.0000001);
    cudaDeviceSynchronize();
    fns[op]<<<1, 32>>>(out, outf, iters, cyc, 1.0000001);
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    *cycles_per_op = static_cast<double>(h) / (16.0 * iters);
    cudaFree(out); cudaFree(outf); cudaFree(cyc);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// ---- row-staging probe: how fast can one-warp CTAs move rows into registers?
// Each CTA (one warp) processes `steps` rows of `row_bytes`, the next row index
// depending on the data of the current one (the construction's dependence).
//   mode 0: TMA (cp.async.bulk) into smem, mbarrier wait, LDS.128 + sum
//   mode 1: same, but the next row's TMA is issued before the reads (2 buffers)
//   mode 2: LDG.128 (ld.global.nc) straight into registers + sum
//   mode 3: LDS.128 + sum of a resident smem row (no refill)
//   mode 4: LDG.128 with L1::no_allocate
namespace {
__device__ __forceinline__ uint32_t pr_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void pr_tma(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pr_smem(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            pr_smem(dst)),
        "l"(src), "r"(bytes), "r"(pr_smem(bar))
        : "memory");
}
__device__ __forceinline__ void pr_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
            pr_smem(bar)),
        "r"(phase)
        : "memory");
}
template <int MODE, int NV>
__global__ void __launch_bounds__(32, MODE == 6 ? 8 : 17) k_stage(const float4* __restrict__ rows, int nrows, int steps,
                                                  float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    float4* buf0 = reinterpret_cast<float4*>(sm + 128);
    float4* buf1 = buf0 + 32 * NV;
    const int lane = threadIdx.x;
    constexpr uint32_t RB = 32 * NV * 16;
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(pr_smem(bar)));
    __syncwarp();
    uint32_t phase = 0;
    uint32_t h = blockIdx.x * 2654435761u + 12345u;
    int idx = h % nrows;
    float acc = 0.f;
    if (MODE == 1 || MODE == 3) {
        if (lane == 0) pr_tma(buf0, rows + static_cast<size_t>(idx) * 32 * NV, RB, bar);
        pr_wait(bar, phase);
        phase ^= 1;
    }
    int cb = 0;
    for (int s = 0; s < steps; ++s) {
        h = h * 1664525u + 1013904223u;
        float4* cur = (MODE == 1 && cb) ? buf1 : buf0;
        if (MODE == 0) {
            __syncwarp();
            if (lane == 0) pr_tma(buf0, rows + static_cast<size_t>(idx) * 32 * NV, RB, bar);
            pr_wait(bar, phase);
            phase ^= 1;
        }
        if (MODE == 5) { // the same row as 4 bulk copies (one per lane 0..3)
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pr_smem(bar)),
                             "r"(RB)
                             : "memory");
            __syncwarp();
            if (lane < 4) {
                const uint32_t q = RB / 4;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        pr_smem(reinterpret_cast<char*>(buf0) + lane * q)),
                    "l"(reinterpret_cast<const char*>(rows + static_cast<size_t>(idx) * 32 * NV) + lane * q),
                    "r"(q), "r"(pr_smem(bar))
                    : "memory");
            }
            pr_wait(bar, phase);
            phase ^= 1;
        }
        if (MODE == 6) { // LDG, two rows in flight (data-independent index)
            float4 a[NV], b[NV];
            const float4* g0 = rows + static_cast<size_t>(idx) * 32 * NV;
#pragma unroll
            for (int t = 0; t < NV; ++t) a[t] = __ldg(g0 + t * 32 + lane);
            for (; s + 1 < steps; s += 2) {
                h = h * 1664525u + 1013904223u;
                const float4* g1 = rows + static_cast<size_t>((h >> 8) % nrows) * 32 * NV;
#pragma unroll
                for (int t = 0; t < NV; ++t) b[t] = __ldg(g1 + t * 32 + lane);
                float s0 = 0.f;
#pragma unroll
                for (int t = 0; t < NV; ++t) s0 += (a[t].x + a[t].y) + (a[t].z + a[t].w);
                h = h * 1664525u + 1013904223u;
                const float4* g2 = rows + static_cast<size_t>((h >> 8) % nrows) * 32 * NV;
#pragma unroll
                for (int t = 0; t < NV; ++t) a[t] = __ldg(g2 + t * 32 + lane);
#pragma unroll
                for (int t = 0; t < NV; ++t) s0 += (b[t].x + b[t].y) + (b[t].z + b[t].w);
                acc += s0;
            }
            break;
        }
        float sum = 0.f;
        const float4* g = rows + static_cast<size_t>(idx) * 32 * NV;
        if (MODE == 1) { // next row index is data-independent here (best case)
            const int nidx = (h >> 8) % nrows;
            __syncwarp();
            if (lane == 0) pr_tma(cb ? buf0 : buf1, rows + static_cast<size_t>(nidx) * 32 * NV, RB, bar);
            idx = nidx;
        }
#pragma unroll
        for (int t = 0; t < NV; ++t) {
            float4 v;
            if (MODE == 2) v = __ldg(g + t * 32 + lane);
            else if (MODE == 4) {
                asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                             : "l"(g + t * 32 + lane));
            } else if (MODE == 3) {
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                             : "r"(pr_smem(cur + t * 32 + lane)));
            } else v = cur[t * 32 + lane];
            sum += (v.x + v.y) + (v.z + v.w);
        }
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        acc += sum;
        if (MODE == 1) {
            pr_wait(bar, phase);
            phase ^= 1;
            cb ^= 1;
        } else {
            idx = static_cast<int>((h >> 8) % nrows) + static_cast<int>(sum); // data-dependent
            if (idx >= nrows) idx = 0;
        }
    }
    if (acc == 1234.5f) *sink = acc;
}
template <int MODE>
int run_stage(int device, int warps_per_sm, int steps, double* gbps, double* ms_out) {
    constexpr int NV = 19;
    constexpr int RB = 32 * NV * 16;
    const int nrows = 2392;
    float4* rows = nullptr;
    float* sink = nullptr;
    if (cudaMalloc(&rows, static_cast<size_t>(nrows) * RB) != cudaSuccess) return 2;
    cudaMalloc(&sink, 4);
    cudaMemset(rows, 0, static_cast<size_t>(nrows) * RB);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int smem = 128 + RB * ((MODE == 1) ? 2 : 1);
    cudaFuncSetAttribute(k_stage<MODE, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * warps_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_stage<MODE, NV><<<grid, 32, smem>>>(rows, nrows, 50, sink);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k_stage<MODE, NV><<<grid, 32, smem>>>(rows, nrows, steps, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms;
    *gbps = static_cast<double>(grid) * steps * RB / (ms * 1e-3) / 1e9;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(rows);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
} // namespace

extern "C" int aco_probe_stage(int device, int mode, int warps_per_sm, int steps, double* gbps,
                               double* ms) {
    cudaSetDevice(device);
    switch (mode) {
    case 0: return run_stage<0>(device, warps_per_sm, steps, gbps, ms);
    case 1: return run_stage<1>(device, warps_per_sm, steps, gbps, ms);
    case 2: return run_stage<2>(device, warps_per_sm, steps, gbps, ms);
    case 3: return run_stage<3>(device, warps_per_sm, steps, gbps, ms);
    case 4: return run_stage<4>(device, warps_per_sm, steps, gbps, ms);
    case 5: return run_stage<5>(device, warps_per_sm, steps, gbps, ms);
    default: return run_stage<6>(device, warps_per_sm, steps, gbps, ms);
    }
}

// ---------------------------------------------------------------------------
// Cluster / DSMEM latencies (a thread-block
// cluster per ant).  One warp per CTA, a cluster of K CTAs on K SMs:
//   mode 0: DSMEM ping-pong between CTA 0 and CTA 1 (st.shared::cluster into
//           the peer's flag, spin on the own flag) — cycles per ROUND TRIP;
//   mode 1: cluster.sync() back to back — cycles per barrier;
//   mode 2: the per-step exchange a cluster-per-ant roulette needs: every CTA
//           writes its partial row total into every CTA's slot, one
//           cluster.sync(), every CTA folds the K partials — cycles per step.
#include <cooperative_groups.h>
namespace cgx = cooperative_groups;

template <int K>
__global__ void __cluster_dims__(K, 1, 1) k_cluster_probe(int mode, int iters, long long* out) {
    __shared__ volatile unsigned flag;
    __shared__ double part[16];
    cgx::cluster_group cl = cgx::this_cluster();
    const unsigned r = cl.block_rank();
    if (threadIdx.x == 0) flag = 0;
    for (int k = threadIdx.x; k < 16; k += 32) part[k] = 0.0;
    cl.sync();
    long long t0 = clock64();
    double acc = 0.0;
    if (mode == 0) {
        if (threadIdx.x == 0 && r < 2) {
            volatile unsigned* peer = cl.map_shared_rank(const_cast<unsigned*>(&flag), r ^ 1u);
            for (int i = 1; i <= iters; ++i) {
                if (r == 0) {
                    *peer = i;
                    while (flag != static_cast<unsigned>(i)) {}
                } else {
                    while (flag != static_cast<unsigned>(i)) {}
                    *peer = i;
                }
            }
        }
    } else if (mode == 1) {
        for (int i = 0; i < iters; ++i) cl.sync();
    } else {
        for (int i = 0; i < iters; ++i) {
            const double mine = static_cast<double>(r + i);
            if (threadIdx.x < K) {
                double* dst = cl.map_shared_rank(part, threadIdx.x);
                dst[(i & 1) * 8 + r] = mine;
            }
            cl.sync();
            double s = 0.0;
            for (int k = 0; k < K; ++k) s += part[(i & 1) * 8 + k];
            acc += s;
        }
    }
    const long long t1 = clock64();
    cl.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = static_cast<long long>(acc);
    }
}

extern "C" int aco_probe_cluster(int device, int K, int mode, int iters, double* cycles_per_iter) {
    cudaSetDevice(device);
    long long* d = nullptr;
    cudaMalloc(&d, 2 * sizeof(long long));
    if (K == 2) k_cluster_probe<2><<<2, 32>>>(mode, iters, d);
    else if (K == 4) k_cluster_probe<4><<<4, 32>>>(mode, iters, d);
    else k_cluster_probe<8><<<8, 32>>>(mode, iters, d);
    long long h[2] = {0, 0};
    const cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return 1;
    *cycles_per_iter = static_cast<double>(h[0]) / iters;
    return 0;
}

// ---- TMA row copy: issue cost and completion latency of one 10 KB row as
// K bulk copies on one mbarrier, one warp alone on the GPU (the chain the
// latency-bound construction launches pay per step).  mode 0: issued by lane
// 0 inside a divergent branch (as the kernel does); mode 1: the same from a
// warp-uniform address after elect.  Per iteration: rows[i % nrows].
__global__ void k_tma_probe(const float* __restrict__ rows, int nrows, int row_floats, int K, int mode,
                            int iters, long long* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    float* buf = reinterpret_cast<float*>(sm + 128);
    const int lane = threadIdx.x & 31;
    const uint32_t sbar = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    const uint32_t sbuf = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t bytes = static_cast<uint32_t>(row_floats * 4);
    const uint32_t piece = ((bytes / K) + 15u) & ~15u;
    long long t_issue = 0, t_total = 0;
    uint32_t phase = 0;
    float sink = 0.f;
    for (int it = 0; it < iters; ++it) {
        const float* src = rows + static_cast<size_t>((it * 7919) % nrows) * row_floats;
        __syncwarp();
        // mode: 0 fence + expect_tx + copies; 1 expect_tx + copies (no proxy
        // fence, as the kernel's speculative refill); 2 copies only (the
        // expect_tx before the timed window)
        if (mode == 2 && lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes)
                         : "memory");
        __syncwarp();
        const long long t0 = clock64();
        if (lane == 0) {
            {
                if (mode == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (mode <= 1)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes)
                                 : "memory");
                for (uint32_t off = 0; off < bytes; off += piece) {
                    const uint32_t b = bytes - off < piece ? bytes - off : piece;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            sbuf + off),
                        "l"(reinterpret_cast<const char*>(src) + off), "r"(b), "r"(sbar)
                        : "memory");
                }
            }
        }
        __syncwarp();
        const long long t1 = clock64();
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "W_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra W_%=;\n}" ::"r"(sbar),
            "r"(phase)
            : "memory");
        phase ^= 1u;
        sink += buf[lane * 37 % row_floats];
        const long long t2 = clock64();
        t_issue += t1 - t0;
        t_total += t2 - t0;
    }
    if (lane == 0) {
        out[0] = t_issue;
        out[1] = t_total;
        out[2] = static_cast<long long>(sink);
    }
}

extern "C" int aco_probe_tma(int device, int row_floats, int K, int mode, int iters, double* issue_cycles,
                             double* total_cycles) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    const int nrows = 2048;
    float* rows = nullptr;
    long long* out = nullptr;
    cudaMalloc(&rows, static_cast<size_t>(nrows) * row_floats * sizeof(float));
    cudaMemset(rows, 0, static_cast<size_t>(nrows) * row_floats * sizeof(float));
    cudaMalloc(&out, 3 * sizeof(long long));
    const size_t smem = 128 + static_cast<size_t>(row_floats) * 4;
    cudaFuncSetAttribute(k_tma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    // warm L2 with a first pass, then time
    k_tma_probe<<<1, 32, smem>>>(rows, nrows, row_floats, K, mode, nrows, out);
    k_tma_probe<<<1, 32, smem>>>(rows, nrows, row_floats, K, mode, iters, out);
    long long h[3] = {0, 0, 0};
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    const int rc = cudaGetLastError() == cudaSuccess ? 0 : 2;
    *issue_cycles = static_cast<double>(h[0]) / iters;
    *total_cycles = static_cast<double>(h[1]) / iters;
    cudaFree(rows);
    cudaFree(out);
    return rc;
}
