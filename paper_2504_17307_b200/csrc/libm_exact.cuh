// libm_exact.cuh -- device restatement of the two libm calls CUBIC makes
// (reference src/cc.cpp:60 and :93 std::cbrt, :63 std::pow(t - k, 3)),
// bit-identical to the host's glibc 2.39 (Ubuntu 2.39-0ubuntu8.5):
//
//  * cbrt: sysdeps/ieee754/dbl-64/s_cbrt.c (frexp reduction, degree-6
//    polynomial, one rational Halley step, factor[2 + xe % 3], ldexp);
//    built for baseline x86-64, so no operation is contracted.
//  * pow: sysdeps/ieee754/dbl-64/e_pow.c (log_inline in double-double, then
//    exp_inline with a 2^(k/128) table), as dispatched on an FMA/AVX2 host
//    (the e_pow-fma.c ifunc variant: __FP_FAST_FMA paths plus GCC's
//    contraction of a*b+c where the product has a single use in the same
//    basic block).  Tables: libm_tables.h (tools/gen_libm_tables.py).
//
// Every operation is an explicit round-to-nearest intrinsic so nvcc cannot
// contract or reorder.  Verified against the host libm on 2e8 inputs (all
// exponent ranges, both signs) in the CPU restatement and on the device by
// tests/test_cubic_gpu.py::test_libm_restatement_matches_host.
#pragma once
#include <stdint.h>

#include "libm_tables.h"

namespace cnb {

__device__ __forceinline__ double as_d(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
__device__ __forceinline__ uint64_t as_u(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }

// s_cbrt.c: factor[] = {1/SQR_CBRT2, 1/CBRT2, 1, CBRT2, SQR_CBRT2}, the
// divisions folded by the compiler (correctly rounded)
__device__ __forceinline__ double libm_cbrt(double x) {
    const uint64_t ux = as_u(x);
    const uint64_t ax = ux & 0x7fffffffffffffffull;
    if (ax == 0 || ax >= 0x7ff0000000000000ull) return __dadd_rn(x, x);  // zero, inf, nan
    // frexp(|x|) -> xm in [0.5, 1), xe (subnormals normalised first)
    int xe;
    uint64_t m = ax;
    if ((ax >> 52) == 0) {
        const double s = __dmul_rn(as_d(ax), 0x1p54);
        m = as_u(s);
        xe = static_cast<int>(m >> 52) - 1022 - 54;
    } else {
        xe = static_cast<int>(ax >> 52) - 1022;
    }
    const double xm = as_d((m & 0x000fffffffffffffull) | 0x3fe0000000000000ull);
    double u = __dsub_rn(0.784932344976639262, __dmul_rn(0.145263899385486377, xm));
    u = __dmul_rn(__dadd_rn(-1.83469277483613086, __dmul_rn(u, xm)), xm);
    u = __dmul_rn(__dadd_rn(2.44693122563534430, u), xm);
    u = __dmul_rn(__dadd_rn(-2.11499494167371287, u), xm);
    u = __dmul_rn(__dadd_rn(1.50819193781584896, u), xm);
    u = __dadd_rn(0.354895765043919860, u);
    const double t2 = __dmul_rn(__dmul_rn(u, u), u);
    const double num = __dadd_rn(t2, __dmul_rn(2.0, xm));
    const double den = __dadd_rn(__dmul_rn(2.0, t2), xm);
    const int fi = xe % 3;
    const double f = fi == -2 ? 0x1.428a2f98d728ap-1 : fi == -1 ? 0x1.965fea53d6e3cp-1 : fi == 0 ? 1.0
                     : fi == 1 ? 0x1.428a2f98d728bp+0 : 0x1.965fea53d6e3dp+0;
    double ym = __dmul_rn(__ddiv_rn(__dmul_rn(u, num), den), f);
    // ldexp(±ym, xe / 3): |ym| in (0.5, 2), exponent change stays normal for
    // every finite input (cube roots of doubles are within [2^-358, 2^342])
    const int sc = xe / 3;
    ym = as_d(as_u(ym) + (static_cast<uint64_t>(static_cast<int64_t>(sc)) << 52));
    return x > 0.0 ? ym : -ym;
}

// e_pow.c exp_inline's specialcase (|x| >= 512): scale may over/underflow
__device__ __forceinline__ double libm_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ull) == 0) {
        sbits -= 1009ull << 52;
        const double scale = as_d(sbits);
        return __dmul_rn(0x1p1009, __fma_rn(scale, tmp, scale));
    }
    sbits += 1022ull << 52;
    const double scale = as_d(sbits);
    const double st = __dmul_rn(scale, tmp);  // two uses in two blocks: not contracted
    double y = __dadd_rn(scale, st);
    if (fabs(y) < 1.0) {
        const double one = y < 0.0 ? -1.0 : 1.0;
        double lo = __dadd_rn(__dsub_rn(scale, y), st);
        const double hi = __dadd_rn(one, y);
        lo = __dadd_rn(__dadd_rn(__dsub_rn(one, hi), y), lo);
        y = __dsub_rn(__dadd_rn(hi, lo), one);
        if (y == 0) y = as_d(sbits & 0x8000000000000000ull);
    }
    return __dmul_rn(0x1p-1022, y);
}

// pow(x, 3.0) (y is an odd integer: the sign of x carries through
// sign_bias).  Finite x only; CUBIC's argument t - K always is.
__device__ __forceinline__ double libm_pow3(double x) {
    const double y = 3.0;
    uint32_t sign_bias = 0;
    uint64_t ix = as_u(x);
    uint32_t topx = static_cast<uint32_t>(ix >> 52);
    if (topx - 0x001u >= 0x7ffu - 0x001u) {
        if (2 * ix - 1 >= 2 * 0x7ff0000000000000ull - 1) {  // zero / inf / nan
            double x2 = __dmul_rn(x, x);
            if (ix >> 63) x2 = -x2;
            return x2;
        }
        if (ix >> 63) {  // finite x < 0, y odd
            sign_bias = 0x800u << 7;
            ix &= 0x7fffffffffffffffull;
            topx &= 0x7ffu;
        }
        if (topx == 0) {  // subnormal
            ix = as_u(__dmul_rn(x, 0x1p52));
            ix &= 0x7fffffffffffffffull;
            ix -= 52ull << 52;
        }
    }
    // log_inline (N = 128, OFF = 0x3fe6955500000000)
    const double Ln2hi = as_d(kPowLogData[0]), Ln2lo = as_d(kPowLogData[1]);
    const uint64_t tmp = ix - 0x3fe6955500000000ull;
    const int i = static_cast<int>((tmp >> (52 - 7)) % 128);
    const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double z = as_d(iz), kd = static_cast<double>(k);
    const double invc = as_d(kPowLogData[9 + 4 * i]), logc = as_d(kPowLogData[9 + 4 * i + 2]),
                 logctail = as_d(kPowLogData[9 + 4 * i + 3]);
    const double r = __fma_rn(z, invc, -1.0);
    const double t1 = __fma_rn(kd, Ln2hi, logc);
    const double t2 = __dadd_rn(t1, r);
    const double lo1 = __fma_rn(kd, Ln2lo, logctail);
    const double lo2 = __dadd_rn(__dsub_rn(t1, t2), r);
    const double A0 = as_d(kPowLogData[2]), A1 = as_d(kPowLogData[3]), A2 = as_d(kPowLogData[4]),
                 A3 = as_d(kPowLogData[5]), A4 = as_d(kPowLogData[6]), A5 = as_d(kPowLogData[7]),
                 A6 = as_d(kPowLogData[8]);
    const double ar = __dmul_rn(A0, r), ar2 = __dmul_rn(r, ar), ar3 = __dmul_rn(r, ar2);
    const double hi = __dadd_rn(t2, ar2);
    const double lo3 = __fma_rn(ar, r, -ar2);
    const double lo4 = __dadd_rn(__dsub_rn(t2, hi), ar2);
    // p = ar3 * (...) has one use, in the sum below: contracted into it
    const double pz = __fma_rn(ar2, __fma_rn(ar2, __fma_rn(r, A6, A5), __fma_rn(r, A4, A3)), __fma_rn(r, A2, A1));
    const double lo = __fma_rn(ar3, pz, __dadd_rn(__dadd_rn(__dadd_rn(lo1, lo2), lo3), lo4));
    const double ly = __dadd_rn(hi, lo);
    const double ltail = __dadd_rn(__dsub_rn(hi, ly), lo);
    // y * log(x) in double-double
    const double ehi = __dmul_rn(y, ly);
    const double elo = __fma_rn(y, ltail, __fma_rn(y, ly, -ehi));
    // exp_inline(ehi, elo, sign_bias)
    uint32_t abstop = static_cast<uint32_t>(as_u(ehi) >> 52) & 0x7ffu;
    const uint32_t t54 = static_cast<uint32_t>(as_u(0x1p-54) >> 52), t512 = static_cast<uint32_t>(as_u(512.0) >> 52),
                   t1024 = static_cast<uint32_t>(as_u(1024.0) >> 52);
    if (abstop - t54 >= t512 - t54) {
        if (abstop - t54 >= 0x80000000u) {
            const double one = __dadd_rn(1.0, ehi);
            return sign_bias ? -one : one;
        }
        if (abstop >= t1024) {  // overflow / underflow
            if (as_u(ehi) >> 63) return sign_bias ? -0.0 : 0.0;
            return sign_bias ? -__longlong_as_double(0x7ff0000000000000ll) : __longlong_as_double(0x7ff0000000000000ll);
        }
        abstop = 0;
    }
    const double InvLn2N = as_d(kExpData[0]), Shift = as_d(kExpData[1]), NegLn2hiN = as_d(kExpData[2]),
                 NegLn2loN = as_d(kExpData[3]);
    const double C2 = as_d(kExpData[4]), C3 = as_d(kExpData[5]), C4 = as_d(kExpData[6]), C5 = as_d(kExpData[7]);
    double ekd = __fma_rn(InvLn2N, ehi, Shift);
    const uint64_t ki = as_u(ekd);
    ekd = __dsub_rn(ekd, Shift);
    double er = __fma_rn(ekd, NegLn2loN, __fma_rn(ekd, NegLn2hiN, ehi));
    er = __dadd_rn(er, elo);
    const uint64_t idx = 2 * (ki % 128);
    const uint64_t top = (ki + sign_bias) << (52 - 7);
    const double etail = as_d(kExpData[22 + idx]);
    const uint64_t sbits = kExpData[22 + idx + 1] + top;
    const double r2 = __dmul_rn(er, er);
    const double etmp =
        __fma_rn(__dmul_rn(r2, r2), __fma_rn(er, C5, C4), __fma_rn(r2, __fma_rn(er, C3, C2), __dadd_rn(etail, er)));
    if (abstop == 0) return libm_exp_special(etmp, sbits, ki);
    const double scale = as_d(sbits);
    return __fma_rn(scale, etmp, scale);
}

}  // namespace cnb
