/* libm_restate.c -- TEST INFRASTRUCTURE ONLY (part of liboracle.so).
 *
 * CPU restatement of the two glibc 2.39 calls the reference's CUBIC makes
 * (src/cc.cpp:60/:93 std::cbrt, :63 std::pow(t - k, 3)):
 *   - cbrt: sysdeps/ieee754/dbl-64/s_cbrt.c (baseline x86-64 build: no FMA);
 *   - pow:  sysdeps/ieee754/dbl-64/e_pow.c as dispatched on an FMA/AVX2 host
 *           (e_pow-fma.c: __FP_FAST_FMA paths plus GCC's contraction of a*b+c
 *           whose product has one use in the same basic block).
 * Tables: paper_2504_17307_b200/csrc/libm_tables.h (extracted from the host
 * libm by tools/gen_libm_tables.py).  orc_libm_host() calls the host libm
 * itself (the reference's own code path) so tests can pin the restatement
 * (tests/test_oracle.py) and the device copy (tests/test_cubic_gpu.py).
 * Compiled with -ffp-contract=off: every fused operation is an explicit fma(). */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../paper_2504_17307_b200/csrc/libm_tables.h"

static uint64_t asu(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static double asd(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

double orc_cbrt(double x) {
    static const double factor[5] = {1.0 / 1.5874010519681994748, 1.0 / 1.2599210498948731648, 1.0,
                                     1.2599210498948731648, 1.5874010519681994748};
    int xe;
    double xm = frexp(fabs(x), &xe);
    if (xe == 0 && fpclassify(x) <= FP_ZERO) return x + x;
    double u = (0.354895765043919860 +
                ((1.50819193781584896 +
                  ((-2.11499494167371287 +
                    ((2.44693122563534430 +
                      ((-1.83469277483613086 + (0.784932344976639262 - 0.145263899385486377 * xm) * xm) * xm)) *
                     xm)) *
                   xm)) *
                 xm));
    double t2 = u * u * u;
    double ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * factor[2 + xe % 3];
    return ldexp(x > 0.0 ? ym : -ym, xe / 3);
}

static double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000) == 0) {
        sbits -= 1009ull << 52;
        double scale = asd(sbits);
        return 0x1p1009 * fma(scale, tmp, scale);
    }
    sbits += 1022ull << 52;
    double scale = asd(sbits);
    double st = scale * tmp;
    double y = scale + st;
    if (fabs(y) < 1.0) {
        double one = y < 0.0 ? -1.0 : 1.0;
        double lo = scale - y + st;
        double hi = one + y;
        lo = one - hi + y + lo;
        y = (hi + lo) - one;
        if (y == 0) y = asd(sbits & 0x8000000000000000ull);
    }
    return 0x1p-1022 * y;
}

double orc_pow3(double x) {
    const double y = 3.0;
    uint32_t sign_bias = 0;
    uint64_t ix = asu(x);
    uint32_t topx = (uint32_t)(ix >> 52);
    if (topx - 0x001 >= 0x7ff - 0x001) {
        if (2 * ix - 1 >= 2 * asu(INFINITY) - 1) {
            double x2 = x * x;
            if (ix >> 63) x2 = -x2;
            return x2;
        }
        if (ix >> 63) {
            sign_bias = 0x800 << 7;
            ix &= 0x7fffffffffffffffull;
            topx &= 0x7ff;
        }
        if (topx == 0) {
            ix = asu(x * 0x1p52);
            ix &= 0x7fffffffffffffffull;
            ix -= 52ull << 52;
        }
    }
    const double* P = (const double*)kPowLogData;
    uint64_t tmp = ix - 0x3fe6955500000000ull;
    int i = (int)((tmp >> (52 - 7)) % 128);
    int k = (int)((int64_t)tmp >> 52);
    uint64_t iz = ix - (tmp & 0xfffull << 52);
    double z = asd(iz), kd = (double)k;
    double invc = P[9 + 4 * i], logc = P[9 + 4 * i + 2], logctail = P[9 + 4 * i + 3];
    double r = fma(z, invc, -1.0);
    double t1 = fma(kd, P[0], logc);
    double t2 = t1 + r;
    double lo1 = fma(kd, P[1], logctail);
    double lo2 = t1 - t2 + r;
    const double* A = P + 2;
    double ar = A[0] * r, ar2 = r * ar, ar3 = r * ar2;
    double hi = t2 + ar2;
    double lo3 = fma(ar, r, -ar2);
    double lo4 = t2 - hi + ar2;
    /* p = ar3 * (...) has one use, in the sum: contracted into it */
    double pz = fma(ar2, fma(ar2, fma(r, A[6], A[5]), fma(r, A[4], A[3])), fma(r, A[2], A[1]));
    double lo = fma(ar3, pz, lo1 + lo2 + lo3 + lo4);
    double ly = hi + lo;
    double ltail = hi - ly + lo;
    double ehi = y * ly;
    double elo = fma(y, ltail, fma(y, ly, -ehi));
    uint32_t abstop = (uint32_t)(asu(ehi) >> 52) & 0x7ff;
    const uint32_t t54 = (uint32_t)(asu(0x1p-54) >> 52), t512 = (uint32_t)(asu(512.0) >> 52),
                   t1024 = (uint32_t)(asu(1024.0) >> 52);
    if (abstop - t54 >= t512 - t54) {
        if (abstop - t54 >= 0x80000000u) {
            double one = 1.0 + ehi;
            return sign_bias ? -one : one;
        }
        if (abstop >= t1024) {
            if (asu(ehi) >> 63) return sign_bias ? -0.0 : 0.0;
            return sign_bias ? -INFINITY : INFINITY;
        }
        abstop = 0;
    }
    const double* E = (const double*)kExpData;
    const uint64_t* T = kExpData + 22;
    double ekd = fma(E[0], ehi, E[1]);
    uint64_t ki = asu(ekd);
    ekd -= E[1];
    double er = fma(ekd, E[3], fma(ekd, E[2], ehi));
    er += elo;
    uint64_t idx = 2 * (ki % 128);
    uint64_t top = (ki + sign_bias) << (52 - 7);
    double etail = asd(T[idx]);
    uint64_t sbits = T[idx + 1] + top;
    double r2 = er * er;
    double etmp = fma(r2 * r2, fma(er, E[7], E[6]), fma(r2, fma(er, E[5], E[4]), etail + er));
    if (abstop == 0) return exp_special(etmp, sbits, ki);
    double scale = asd(sbits);
    return fma(scale, etmp, scale);
}

/* mode 0 cbrt, 1 pow(x, 3.0): restated (restated != 0) or the host libm */
void orc_libm(int mode, int restated, const double* in, double* out, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) {
        if (restated) out[i] = mode == 0 ? orc_cbrt(in[i]) : orc_pow3(in[i]);
        else out[i] = mode == 0 ? cbrt(in[i]) : pow(in[i], 3.0);
    }
}
