// Device Philox4x32-10 keyed by (seed; draw, step, ant, iteration).
// Same permutation, key schedule and 53-bit mantissa extraction as the
// reference RngStream (rng.hpp:12-43 round/permute, :74-80 uniform_at), so
// every draw is bit-identical: the multiply-high/low pairs map to IMAD.HI /
// IMAD and the final (bits >> 11) * 2^-53 is exact in FP64.
#pragma once
#include <cstdint>

namespace acob200 {

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
#endif
}

__host__ __device__ __forceinline__ void philox4x32_10(uint32_t& v0, uint32_t& v1, uint32_t& v2,
                                                       uint32_t& v3, uint64_t key) {
    uint32_t k0 = static_cast<uint32_t>(key);
    uint32_t k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = mulhi32(0xD2511F53u, v0), lo0 = 0xD2511F53u * v0;
        const uint32_t hi1 = mulhi32(0xCD9E8D57u, v2), lo1 = 0xCD9E8D57u * v2;
        const uint32_t n0 = hi1 ^ v1 ^ k0;
        const uint32_t n2 = hi0 ^ v3 ^ k1;
        v0 = n0;
        v1 = lo1;
        v2 = n2;
        v3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__host__ __device__ __forceinline__ double philox_uniform(uint64_t seed, uint32_t iteration,
                                                          uint32_t ant, uint32_t step,
                                                          uint32_t draw) {
    uint32_t v0 = draw, v1 = step, v2 = ant, v3 = iteration;
    philox4x32_10(v0, v1, v2, v3, seed);
    const uint64_t bits = (static_cast<uint64_t>(v1) << 32) | v0;
    return static_cast<double>(bits >> 11) * 0x1.0p-53;
}

} // namespace acob200
