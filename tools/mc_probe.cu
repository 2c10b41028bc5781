// mc_probe.cu — can this box build an NVLS multicast object over ONE device
// and drive multimem.red.add.f64 through it?  (DESIGN §9 f2: round 1 saw
// cuMulticastCreate reject a one-device object; this probes the variants.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/_mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#define CU(x)                                                                  \
    do {                                                                       \
        CUresult r_ = (x);                                                     \
        if (r_ != CUDA_SUCCESS) {                                              \
            const char* s_ = nullptr;                                          \
            cuGetErrorName(r_, &s_);                                           \
            std::printf("  %s -> %s (%d)\n", #x, s_ ? s_ : "?", (int)r_);      \
            return false;                                                      \
        }                                                                      \
    } while (0)

__global__ void k_mm_red(double* mc, int count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const double v = 0.25 * (i % 7);
        asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(mc + i), "d"(v) : "memory");
    }
}
__global__ void k_mm_ld(const double* mc, double* out, int count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        double v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc + i) : "memory");
        out[i] = v;
    }
}

static bool try_variant(CUdevice dev, unsigned long long handle_types, const char* name) {
    std::printf("variant %s\n", name);
    CUmulticastObjectProp mp{};
    mp.numDevices = 1;
    mp.handleTypes = handle_types;
    mp.size = 1 << 21;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    size_t gmin = 0;
    CU(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
    std::printf("  granularity recommended %zu minimum %zu\n", gran, gmin);
    const size_t size = ((size_t(8) << 20) + gran - 1) / gran * gran;
    mp.size = size;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    std::printf("  cuMulticastCreate ok (size %zu)\n", size);
    CU(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)handle_types;
    size_t ag = 0;
    CU(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle phys;
    CU(cuMemCreate(&phys, size, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, phys, 0, size, 0));
    CUdeviceptr uc = 0, mcp = 0;
    CU(cuMemAddressReserve(&uc, size, gran, 0, 0));
    CU(cuMemMap(uc, size, 0, phys, 0));
    CUmemAccessDesc ad{};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = dev;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(uc, size, &ad, 1));
    CU(cuMemAddressReserve(&mcp, size, gran, 0, 0));
    CU(cuMemMap(mcp, size, 0, mc, 0));
    CU(cuMemSetAccess(mcp, size, &ad, 1));
    std::printf("  mapped unicast %p multicast %p\n", (void*)uc, (void*)mcp);
    const int count = 1 << 20;
    cudaMemset((void*)uc, 0, count * sizeof(double));
    k_mm_red<<<148, 256>>>(reinterpret_cast<double*>(mcp), count);
    k_mm_red<<<148, 256>>>(reinterpret_cast<double*>(mcp), count);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("  multimem.red x2: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return false;
    std::vector<double> h(count);
    cudaMemcpy(h.data(), (void*)uc, count * sizeof(double), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < count; ++i)
        if (h[i] != 0.5 * (i % 7)) ++bad;
    std::printf("  unicast view after reds: %d mismatches\n", bad);
    double* out = nullptr;
    cudaMalloc(&out, count * sizeof(double));
    k_mm_ld<<<148, 256>>>(reinterpret_cast<double*>(mcp), out, count);
    e = cudaDeviceSynchronize();
    std::printf("  multimem.ld_reduce: %s\n", cudaGetErrorString(e));
    if (e == cudaSuccess) {
        cudaMemcpy(h.data(), out, count * sizeof(double), cudaMemcpyDeviceToHost);
        bad = 0;
        for (int i = 0; i < count; ++i)
            if (h[i] != 0.5 * (i % 7)) ++bad;
        std::printf("  ld_reduce values: %d mismatches\n", bad);
    }
    // timing: reds through the multicast address vs plain red.global
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) k_mm_red<<<148 * 8, 256>>>(reinterpret_cast<double*>(mcp), count);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("  multimem.red.add.f64: %.1f G ops/s (1M contiguous doubles x10)\n",
                10.0 * count / (ms * 1e-3) / 1e9);
    cudaFree(out);
    return true;
}

int main() {
    cudaFree(0);
    CUdevice dev;
    cuDeviceGet(&dev, 0);
    int mcs = 0, fab = 0, nvls = 0;
    cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    std::printf("MULTICAST_SUPPORTED=%d FABRIC=%d\n", mcs, fab);
    (void)nvls;
    const bool ok1 = try_variant(dev, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, "posix_fd");
    const bool ok2 = ok1 ? true : try_variant(dev, CU_MEM_HANDLE_TYPE_FABRIC, "fabric");
    const bool ok3 = (ok1 || ok2) ? true : try_variant(dev, CU_MEM_HANDLE_TYPE_NONE, "none");
    std::printf("RESULT %s\n", (ok1 || ok2 || ok3) ? "multicast usable on one device" : "no one-device multicast");
    return 0;
}
