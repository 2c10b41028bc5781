// libaco_probe.so — measurement helpers for the roofline denominators
// (not on the product path).  SURVEY §8(d): "measure the L2 bandwidth with a
// read kernel over a resident buffer of ~50% of the L2, 16-byte loads on all
// SMs"; the same kernel over a buffer far larger than L2 gives HBM read BW.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {

__global__ void k_read(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
             i += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const float4 v = __ldg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1234.5f) *sink = acc; // never true for a zero buffer; keeps the loads
}

} // namespace

extern "C" int aco_probe_read_bw(int device, size_t bytes, int reps, int iters, double* gbps,
                                 double* ms_out) {
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
    k_read<<<sms * 8, 512>>>(buf, n4, 1, sink); // warm (L2-resident when it fits)
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int it = 0; it < iters; ++it) {
        cudaEventRecord(a);
        k_read<<<sms * 8, 512>>>(buf, n4, reps, sink);
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
