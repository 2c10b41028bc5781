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
