// Device pow(x, y) that reproduces THIS HOST's glibc pow bit for bit, so
// compute_choice_info's pow(tau, alpha) (model.hpp:167) stays exact for any
// alpha, not only alpha in {0, 1}.
//
// glibc (2.28+) computes pow as exp(y * log(x)) with a 128-entry log table
// and a 2^(k/128) exp table in double-double arithmetic (the ARM
// optimized-routines algorithm); on x86-64 with FMA + AVX2 the ifunc selects
// a build compiled with -mfma, in which GCC contracted specific a*b+c pairs
// into FMAs.  libm_pow below restates that machine code operation by
// operation (each step annotated with the x86 instruction it mirrors:
// vfmadd = one rounding, separate vmul/vadd = two), using the host libm's
// OWN tables, which host_model.cpp reads out of the loaded libm.so at
// context creation (no glibc data is compiled into this repo).  A device
// self-test against the host's std::pow at creation time refuses the alpha
// path (ACO_E_UNSUPPORTED) if the host dispatched another variant.
//
// Domain: x >= +0 finite (pheromone), y > 0 finite (alpha) — everything the
// choice kernel passes; the special cases glibc takes inside that domain
// (x = +0, subnormal x, |y| < 2^-65 or >= 2^63, exp over/underflow, the
// subnormal-result rounding) are all reproduced.
#pragma once
#include <cstdint>

#include "host_model.hpp" // LibmPowTables

namespace acob200 {

__device__ __forceinline__ double libm_pow_special_exp(double tmp, uint64_t sbits, uint64_t ki) {
    // specialcase(): the exponent of 2^k over/underflowed the scale
    if ((ki & 0x80000000ull) == 0) {
        sbits -= 1009ull << 52;                              // add 0xc0f0...
        const double scale = __longlong_as_double(static_cast<long long>(sbits));
        const double y = __fma_rn(scale, tmp, scale);        // vfmadd132sd
        return __dmul_rn(y, 0x1p1009);
    }
    sbits += 1022ull << 52;
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    const double st = __dmul_rn(tmp, scale);                 // vmulsd (not fused here)
    double y = __dadd_rn(scale, st);                         // vaddsd
    if (fabs(y) < 1.0) {
        const double lo0 = __dadd_rn(__dsub_rn(scale, y), st);
        const double one = y < 0.0 ? -1.0 : 1.0;
        const double hi = __dadd_rn(y, one);
        const double lo = __dadd_rn(__dadd_rn(__dsub_rn(one, hi), y), lo0);
        y = __dsub_rn(__dadd_rn(lo, hi), one);
        if (y == 0.0) y = __longlong_as_double(static_cast<long long>(sbits & 0x8000000000000000ull));
    }
    return __dmul_rn(y, 0x1p-1022);
}

__device__ __noinline__ double libm_pow(double x, double y, const LibmPowTables* __restrict__ T) {
    uint64_t ix = static_cast<uint64_t>(__double_as_longlong(x));
    const uint64_t iy = static_cast<uint64_t>(__double_as_longlong(y));
    const uint32_t topx = static_cast<uint32_t>(ix >> 52);
    const uint32_t topy = static_cast<uint32_t>(iy >> 52) & 0x7ff;
    const bool y_in_range = (topy - 0x3beu) <= 0x7fu; // 2^-65 <= |y| < 2^63
    if (topx - 1u >= 0x7feu) {                         // x == +0 or subnormal (x >= 0 here)
        if (ix == 0) return __dmul_rn(x, x);           // pow(+0, y > 0) = +0
        if (y_in_range) {                              // normalise the subnormal
            ix = static_cast<uint64_t>(__double_as_longlong(__dmul_rn(x, 0x1p52)));
            ix &= 0x7fffffffffffffffull;
            ix -= 52ull << 52;
        }
    } else if (!y_in_range && ix == 0x3ff0000000000000ull) {
        return 1.0;
    }
    if (!y_in_range) {
        if (topy > 0x3bdu)                                 // |y| >= 2^63
            return ix <= 0x3ff0000000000000ull ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
        return ix <= 0x3ff0000000000000ull ? __dsub_rn(1.0, y) : __dadd_rn(y, 1.0); // |y| < 2^-65
    }

    // ---- log_inline (FMA build)
    const uint64_t tmpi = ix - 0x3fe6955500000000ull;
    const int i = static_cast<int>((tmpi >> 45) & 0x7f);
    const int k = static_cast<int>(static_cast<int64_t>(tmpi) >> 52);
    const uint64_t iz = ix - (tmpi & 0xfff0000000000000ull);
    const double z = __longlong_as_double(static_cast<long long>(iz));
    const double kd = static_cast<double>(k);
    const double invc = T->ltab[4 * i], logc = T->ltab[4 * i + 2], logctail = T->ltab[4 * i + 3];
    const double r = __fma_rn(z, invc, -1.0);                 // vfmadd132sd
    const double t1 = __fma_rn(kd, T->ln2hi, logc);           // vfmadd213sd (contracted)
    const double lo1 = __fma_rn(kd, T->ln2lo, logctail);      // vfmadd213sd (contracted)
    const double t2 = __dadd_rn(r, t1);
    const double lo2 = __dadd_rn(__dsub_rn(t1, t2), r);
    const double ar = __dmul_rn(r, T->A[0]);
    const double ar2 = __dmul_rn(r, ar);
    const double ar3 = __dmul_rn(r, ar2);
    const double hi = __dadd_rn(t2, ar2);
    const double lo3 = __fma_rn(ar, r, -ar2);                 // vfmsub132sd
    const double lo4 = __dadd_rn(__dsub_rn(t2, hi), ar2);
    const double p1 = __fma_rn(r, T->A[2], T->A[1]);
    const double p3 = __fma_rn(r, T->A[4], T->A[3]);
    const double p5 = __fma_rn(r, T->A[6], T->A[5]);
    const double q = __fma_rn(ar2, __fma_rn(p5, ar2, p3), p1);
    double lo = __dadd_rn(__dadd_rn(__dadd_rn(lo1, lo2), lo3), lo4);
    lo = __fma_rn(ar3, q, lo);                                // vfmadd231sd (p contracted)
    const double lhi = __dadd_rn(hi, lo);
    const double ltail = __dadd_rn(__dsub_rn(hi, lhi), lo);

    // ---- y * log(x) as ehi + elo
    const double ehi = __dmul_rn(y, lhi);
    const double elo = __fma_rn(y, ltail, __fma_rn(lhi, y, -ehi));
    uint32_t abstop = static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(ehi)) >> 52) & 0x7ff;
    if (abstop - 0x3c9u > 0x3eu) {
        if (static_cast<int>(abstop - 0x3c9u) < 0) return __dadd_rn(ehi, 1.0); // |ehi| < 2^-54
        if (abstop > 0x408u)                                                      // |ehi| >= 1024
            return ehi < 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
        abstop = 0; // 512 <= |ehi| < 1024: the scale needs specialcase()
    }

    // ---- exp_inline (FMA build), sign_bias = 0
    double kd2 = __fma_rn(ehi, T->invln2N, T->shift);         // vfmadd132sd (z + Shift contracted)
    const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd2));
    kd2 = __dsub_rn(kd2, T->shift);
    double er = __fma_rn(kd2, T->negln2hiN, ehi);
    er = __fma_rn(kd2, T->negln2loN, er);
    const int idx = 2 * static_cast<int>(ki & 0x7f);
    const uint64_t top = ki << 45;
    const double tail = __longlong_as_double(static_cast<long long>(T->etab[idx]));
    const uint64_t sbits = T->etab[idx + 1] + top;
    er = __dadd_rn(elo, er);
    const double c23 = __fma_rn(er, T->C[1], T->C[0]);
    const double t_r = __dadd_rn(er, tail);
    const double r2 = __dmul_rn(er, er);
    const double c45 = __fma_rn(er, T->C[3], T->C[2]);
    const double u = __fma_rn(c23, r2, t_r);
    const double r4 = __dmul_rn(r2, r2);
    const double tmp = __fma_rn(c45, r4, u);
    if (abstop == 0) return libm_pow_special_exp(tmp, sbits, ki);
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    return __fma_rn(tmp, scale, scale);                       // vfmadd132sd
}

} // namespace acob200
