// smc_fastmath.h -- fp64 log / cos for the Box-Muller transform and the
// t-likelihood of the PF move kernel (the kernel is FP64/INT issue bound:
// libdevice log and cos cost ~3 and ~2.4 ps per call on B200, these ~half).
//
// Accuracy (tests/test_fastmath.py, against glibc on 4e6+ inputs): log <= 0.52 ulp,
// cos <= 1 ulp -- the same class as glibc/libdevice, so GPU normals stay within a
// few ulp of the reference's (rng.py:85-91).  Header-only and host-compilable so
// the CPU test runs the identical code.
//
// log(x) = k ln2 + log(c_i) + log1p(r),  x = 2^k z,  z in [0.6875, 1.375),
//          k ln2 + log(c_i) exact as a double (table on the 2^-42 grid of LN2_HI),
//          r = z/c_i - 1 via one FMA (|r| <= 2^-10, 512 intervals), c_i = 1 exactly
//          around z = 1 so that r = z - 1 is exact there (full relative accuracy near
//          x = 1), log1p(r) - r by a degree-6 Taylor polynomial (truncation < 2^-63 |r|).
// cos_bm(x), 0 <= x < 8 (x = fl(2 pi u) in Box-Muller): branch-free quadrant
//          reduction, then minimax polynomials on |r| <= pi/4 (coefficients:
//          fdlibm's published __kernel_cos/__kernel_sin constants; see cos_bm).
#pragma once
#ifdef __CUDACC_RTC__  // run-time compiled user kernels (NVRTC has no libc headers)
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef int int32_t;
#ifndef INFINITY
#define INFINITY __longlong_as_double(0x7ff0000000000000LL)
#endif
#else
#include <stdint.h>
#include <string.h>
#include <math.h>
#endif

#ifdef __CUDACC__
#define SMC_HD __host__ __device__ __forceinline__
#define SMC_HDM __host__ __device__ __forceinline__
#define SMC_TABLE __device__ const
#define SMC_CONSTANT __constant__
#else
#define SMC_HD static inline
#define SMC_HDM inline
#define SMC_CONSTANT static const
#define SMC_TABLE static const
#endif

namespace smc_fm {

struct alignas(16) LogEntry {
    double logc_hi;       // -log(invc) on the 2^-42 grid
    float invc, logc_lo;  // 1/c in single precision (exact as a double), the |lo| <= 2^-43 rest
};                        // 16 bytes: one 128-bit load per lookup

SMC_TABLE LogEntry kLogTab[512] = {
#include "smc_logtab.inc"
};

// Constants with non-zero low words live in the constant bank, so each FP64
// instruction takes them as a c[][] operand (as literals they cost two UMOVs
// per use in the issue stream).
SMC_CONSTANT double kLogK[6] = {0x1.2492492492492p-3, -0x1.5555555555555p-3, 0x1.999999999999ap-3,
                                0x1.5555555555555p-2, 0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45};

SMC_HD uint64_t bits(double x)
{
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
SMC_HD double from_bits(uint64_t u)
{
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}
SMC_HD double fma_(double a, double b, double c)
{
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

SMC_HD const LogEntry &log_entry(int i)
{
    return kLogTab[i];
}

// Natural log of a positive normal finite double (precondition; no check).  `tab`: an
// optional shared-memory copy of kLogTab (kernels that stage it), else the global table.
SMC_HD double log_core(double x, const LogEntry *tab = nullptr)
{
    const uint64_t ix = bits(x);
    const uint64_t OFF = 0x3fe6000000000000ull;
    const uint64_t tmp = ix - OFF;
    const int i = (int)((tmp >> 43) & 511);
    const int64_t k = (int64_t)tmp >> 52;
    const double z = from_bits(ix - (tmp & (0xfffull << 52)));
#ifdef __CUDA_ARCH__
    const double2 e = tab ? reinterpret_cast<const double2 *>(tab)[i]
                          : __ldg(reinterpret_cast<const double2 *>(&kLogTab[i]));
    const uint64_t w1 = (uint64_t)__double_as_longlong(e.y);
    const double lhi = e.x, invc = (double)__uint_as_float((uint32_t)w1), llo = (double)__uint_as_float((uint32_t)(w1 >> 32));
#else
    const double invc = kLogTab[i].invc, lhi = kLogTab[i].logc_hi, llo = kLogTab[i].logc_lo;  // float -> double exact
#endif
    const double r = fma_(z, invc, -1.0);
    const double kd = (double)k;
    const double LN2_HI = kLogK[4], LN2_LO = kLogK[5];
    // hi + lo = k ln2 + log c + r with error-free sums: k LN2_HI is exact (42 + 11 bits)
    // and so is w = k LN2_HI + logc_hi (the table puts logc_hi on LN2_HI's 2^-42 grid,
    // tools/gen_logtab.py); hi = w + r is split by Fast2Sum (|w| >= |r| or w = 0)
    const double w = fma_(kd, LN2_HI, lhi);
    const double hi = w + r;
    const double he = r - (hi - w);
    const double lo = he + fma_(kd, LN2_LO, llo);
    // log1p(r) - r = r^2 (-1/2 + r (1/3 + r (-1/4 + r (1/5 - r/6)))), |r| <= 2^-10
    double p = fma_(r, kLogK[1], kLogK[2]);
    p = fma_(r, p, -0.25);
    p = fma_(r, p, kLogK[3]);
    p = fma_(r, p, -0.5);
    return hi + fma_(r * r, p, lo);
}

// Natural log; inputs that are not positive normal finite doubles go to libm.
SMC_HD double log(double x)
{
    // positive normal finite: exponent field in [1, 2046]
    return (bits(x) >> 52) - 1u < 2046u ? log_core(x) : ::log(x);
}

// cos(x) for 0 <= x < 8, BRANCH-FREE (the Box-Muller argument x = fl(2 pi u),
// rng.py:91): one polynomial evaluation whose coefficients are picked by the
// quadrant from a 4-row table, so a warp never diverges and the whole
// normal is one basic block the scheduler can interleave with the Philox work.
//   j = rint(x 2/pi) (shifter: the integer lands in the low word), r = x - j pi/2
//   with pi/2 = C1 + C2 (C1 = fl(pi/2); x - j C1 is exact for x >= pi/4 and j = 0
//   below, the C2 product is folded in by one FMA), z = r^2;
//   even j: cos r = 1 + z (-1/2 + z C(z)),  odd j: sin r = r + (r z) S(z)
//   (fdlibm's __kernel_cos / __kernel_sin minimax coefficients on |r| <= pi/4),
//   and the sign of quadrant j: cos(j pi/2 + r) = A + (z A) p(z) with A = +-1 (even j)
//   or +-r (odd j), A = fma(a1, r, a0) from the (j mod 4) table row.  <= 1.5 ulp
//   (tests/test_fastmath.py), the class of libdevice's cos (2 ulp).
struct alignas(16) CosPoly {
    double a0, a1, q[8];  // A = a1 r + a0; q[7] = 0 pads the row to 5 x 16 bytes
};
#define SMC_COS_Q {-0.5, 4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05, \
                   -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11, 0.0}
#define SMC_SIN_Q {-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04, \
                   2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10, 0.0, 0.0}
SMC_TABLE CosPoly kCosPoly[4] = {
    {1.0, 0.0, SMC_COS_Q},    // j = 0 mod 4:  cos r
    {0.0, -1.0, SMC_SIN_Q},   // j = 1:       -sin r
    {-1.0, 0.0, SMC_COS_Q},   // j = 2:       -cos r
    {0.0, 1.0, SMC_SIN_Q},    // j = 3:        sin r
};
#undef SMC_COS_Q
#undef SMC_SIN_Q
SMC_CONSTANT double kCosK[4] = {0x1.45f306dc9c883p-1, 0x1.921fb54442d18p+0, 0x1.1a62633145c07p-54, 0.0};

SMC_HD double cos_bm(double x, const CosPoly *tab = nullptr)  // tab: optional shared-memory copy
{
    const double SH = 0x1.8p52;
    const double kd = fma_(x, kCosK[0], SH);  // x 2/pi rounded to an integer
    const uint32_t j = (uint32_t)bits(kd);
    const double jd = kd - SH;
    const double r = fma_(-jd, kCosK[2], fma_(-jd, kCosK[1], x));
    const double z = r * r;
#ifdef __CUDA_ARCH__
    double2 a, q01, q23, q45, q67;
    if (tab) {
        const double2 *t = reinterpret_cast<const double2 *>(&tab[j & 3]);
        a = t[0], q01 = t[1], q23 = t[2], q45 = t[3], q67 = t[4];
    } else {
        const double2 *t = reinterpret_cast<const double2 *>(&kCosPoly[j & 3]);
        a = __ldg(t), q01 = __ldg(t + 1), q23 = __ldg(t + 2), q45 = __ldg(t + 3), q67 = __ldg(t + 4);
    }
#else
    const CosPoly &e = kCosPoly[j & 3];
    const struct { double x, y; } a{e.a0, e.a1}, q01{e.q[0], e.q[1]}, q23{e.q[2], e.q[3]}, q45{e.q[4], e.q[5]},
        q67{e.q[6], e.q[7]};
#endif
    double p = fma_(z, q67.x, q45.y);
    p = fma_(z, p, q45.x);
    p = fma_(z, p, q23.y);
    p = fma_(z, p, q23.x);
    p = fma_(z, p, q01.y);
    p = fma_(z, p, q01.x);
    const double A = fma_(a.y, r, a.x);  // exact: +-1 or +-r
    return fma_(z * A, p, A);
}

// sqrt(v) for v = 0 or v in [2^-60, 2^60] (the Box-Muller radius -2 log(1 - u),
// rng.py:91), branch- and select-free: the hardware fp64 rsqrt seed (MUFU.RSQ64H,
// ~2^-22) of v + 2^-1000 (= v unless v = 0, where it keeps the seed finite so the
// root comes out as 0 * y = 0) refined by one Newton step on the reciprocal root
// and one correction of the root itself (the residual v - s^2 by FMA).  Correctly
// rounded except in rare near-halfway cases (<= 1 ulp).
SMC_HD double sqrt_bm(double v)
{
    const double vp = v + 0x1p-1000;
#ifdef __CUDA_ARCH__
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(vp));
#else
    double y = from_bits(bits(1.0 / ::sqrt(vp)) & 0xffffffffe0000000ull);  // a ~fp32-accurate seed, as on the device
#endif
    y = y * fma_(-0.5 * vp * y, y, 1.5);
    const double s = v * y;
    const double d = fma_(-s, s, v);
    return fma_(d, 0.5 * y, s);
}

// a / 10 rounded to nearest, division-free (Markstein): q = a fl(1/10), the exact residual
// a - 10 q by FMA, one correction.  Identical to the IEEE quotient for every a whose quotient
// is normal (tests/test_fastmath.py; below that the PF's t-likelihood only meets it as
// 1 + q = 1).  a = inf gives inf (the NaN of the correction is discarded), NaN stays NaN.
SMC_HD double div10(double a)
{
    const double q = a * 0.1;
    const double r = fma_(-q, 10.0, a);
    const double q1 = fma_(r, 0.1, q);
    return q1 != q1 ? q : q1;
}

// exp(x) for the GMM likelihood (smc_gmm.cu).  x = (128 m + j) ln2/128 + r with
// |r| <= ln2/256; exp(r) - 1 by a degree-5 Taylor polynomial (truncation
// < 2^-60); 2^(j/128) as hi + lo from kExpTab.  Subnormal results are scaled in
// two steps; overflow gives +inf; NaN propagates.  No libm call, no branch.  The table is passed in so the device can
// stage it in shared memory (one LDS.128 per call instead of a global gather).
struct alignas(16) ExpEntry {
    double hi, lo;
};

SMC_TABLE ExpEntry kExpTab[128] = {
#include "smc_exptab.inc"
};

SMC_HD double exp(double x, const ExpEntry *tab)
{
    // Branch-free so that independent calls interleave.  Outside [-746, ln DBL_MAX]
    // the reduction below is garbage and the final selects return 0 / +inf; NaN
    // fails both comparisons and propagates through the arithmetic.
    const double XMAX = 0x1.62e42fefa39efp+9;  // 709.78271289338397 = ln(DBL_MAX) rounded down
    const double SH = 0x1.8p52;
    double kd = fma_(x, 0x1.71547652b82fep+7, SH);
    const int64_t k = (int32_t)(uint32_t)bits(kd);  // round(x 128/ln2) from the shifter's low word
    kd -= SH;
    double r = fma_(-kd, 0x1.62e42fefc0000p-8, x);
    r = fma_(-kd, -0x1.c610ca86c3899p-44, r);
    double p = fma_(r, 1.0 / 120, 1.0 / 24);
    p = fma_(r, p, 1.0 / 6);
    p = fma_(r, p, 0.5);
    p = fma_(r * r, p, r);
    const ExpEntry t = tab[k & 127];
    const double m = fma_(t.hi, p, t.lo) + t.hi;  // 2^(j/128) exp(r), in [1, 2)
    const int64_t e = k >> 7;
    // subnormal results are scaled in two steps so the only rounding is the final multiply
    const bool tiny = e < -1020;
    const double res = from_bits(bits(m) + ((uint64_t)(tiny ? e + 600 : e) << 52)) * (tiny ? 0x1p-600 : 1.0);
    return x < -746.0 ? 0.0 : (x > XMAX ? INFINITY : res);  // exp(-746) rounds to +0
}

// The GMM likelihood's exp: a 256-entry table (2^(j/256), tools/gen_logtab.py) halves the
// reduced argument, |r| <= ln2/512, so a degree-4 polynomial suffices (<= 0.6 ulp,
// tests/test_fastmath.py): one fp64 FMA per call fewer than exp_nonpos (the likelihood's hot loop is fp64-issue
// bound).  Same contract as exp_nonpos (x <= 0, below 2^-1022 flushed to +0); table layout
// (stride, off) as there.
SMC_TABLE ExpEntry kExpTab256[256] = {
#include "smc_exptab256.inc"
};
SMC_HD double exp_nonpos256(double x, const ExpEntry *tab, int stride = 1, int off = 0)
{
    const double SH = 0x1.8p52;
    double kd = fma_(x, 0x1.71547652b82fep+8, SH);  // round(x 256/ln2) in the low word
    const int64_t k = (int32_t)(uint32_t)bits(kd);
    kd -= SH;
    double r = fma_(-kd, 0x1.62e42fefc0000p-9, x);  // ln2/256 hi (35 bits: kd hi exact)
    r = fma_(-kd, -0x1.c610ca86c3899p-45, r);
    // 1/6 + (5/4) h^2 / 120 (h = ln2/512): the r^5/120 term economized into r^3 (max truncation
    // 1.2e-17 instead of 3.8e-17)
    double p = fma_(r, 1.0 / 24, 0x1.555557e54fd54p-3);
    p = fma_(r, p, 0.5);
    p = fma_(r * r, p, r);
    const ExpEntry t = tab[(k & 255) * stride + off];
    const double m = fma_(t.hi, p, t.lo) + t.hi;
    const double res = from_bits(bits(m) + ((uint64_t)(k >> 8) << 52));
    return x < -708.0 ? 0.0 : res;  // -inf included
}

// exp(x) for x <= 0 with the table: no overflow side and no subnormal results
// (below 2^-1022 it flushes to +0) -- for sums whose largest term is exp(0) = 1,
// where anything that small is far below their rounding (the GMM likelihood).
// The constants a DFMA cannot take as an immediate (low mantissa word nonzero): as
// immediates they cost two UMOVs each -- free in a loop that hoists them (the GMM
// likelihood), not in straight-line code evaluating many items (the resampling weights),
// which takes them from the constant bank instead (exp_nonpos_cb: same bits).
SMC_CONSTANT double kExpNpK[8] = {0x1.71547652b82fep+7, 0x1.62e42fefc0000p-8, -0x1.c610ca86c3899p-44,
                                  1.0 / 120, 1.0 / 24, 1.0 / 6, 0.0, 0.0};
// (stride, off): the table may be replicated -- entry k of copy `off` at tab[k stride + off]
// (the GMM kernel keeps 8 copies interleaved so that the 8 lanes of an LDS.128 phase read 8
// different bank groups: no bank conflicts whatever the indices).  Same bits either way.
SMC_HD double exp_nonpos(double x, const ExpEntry *tab, int stride = 1, int off = 0)
{
    const double SH = 0x1.8p52;
    double kd = fma_(x, 0x1.71547652b82fep+7, SH);
    const int64_t k = (int32_t)(uint32_t)bits(kd);
    kd -= SH;
    double r = fma_(-kd, 0x1.62e42fefc0000p-8, x);
    r = fma_(-kd, -0x1.c610ca86c3899p-44, r);
    double p = fma_(r, 1.0 / 120, 1.0 / 24);
    p = fma_(r, p, 1.0 / 6);
    p = fma_(r, p, 0.5);
    p = fma_(r * r, p, r);
    const ExpEntry t = tab[(k & 127) * stride + off];
    const double m = fma_(t.hi, p, t.lo) + t.hi;
    const double res = from_bits(bits(m) + ((uint64_t)(k >> 7) << 52));
    return x < -708.0 ? 0.0 : res;  // -inf included
}

// exp_nonpos with its non-immediate constants from the constant bank (same bits).
SMC_HD double exp_nonpos_cb(double x, const ExpEntry *tab)
{
    const double SH = 0x1.8p52;
    double kd = fma_(x, kExpNpK[0], SH);
    const int64_t k = (int32_t)(uint32_t)bits(kd);
    kd -= SH;
    double r = fma_(-kd, kExpNpK[1], x);
    r = fma_(-kd, kExpNpK[2], r);
    double p = fma_(r, kExpNpK[3], kExpNpK[4]);
    p = fma_(r, p, kExpNpK[5]);
    p = fma_(r, p, 0.5);
    p = fma_(r * r, p, r);
    const ExpEntry t = tab[k & 127];
    const double m = fma_(t.hi, p, t.lo) + t.hi;
    const double res = from_bits(bits(m) + ((uint64_t)(k >> 7) << 52));
    return x < -708.0 ? 0.0 : res;  // -inf included
}

// exp(x) for x <= ~0 without a table (resampling weights W = exp(lw - lse): many
// independent calls per thread, where table lookups congest shared memory / L1):
// x = k ln2 + r, |r| <= ln2/2, exp(r) by its degree-13 Taylor polynomial
// (truncation < 5e-18 relative), coefficients from the constant bank.  Results
// below 2^-1022 (x < -708) flush to +0 -- for a weight that is exactly what its
// quantization floor(W 2^63) gives; x > 708 is outside the contract.
SMC_CONSTANT double kExpPolyK[16] = {
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0,
    1.0 / 40320.0, 1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0,
    0x1.71547652b82fep+0, 0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45, 0.0, 0.0};  // 1/ln2, ln2 hi, lo

SMC_HD double exp_weight(double x)
{
    const double SH = 0x1.8p52;
    double kd = fma_(x, kExpPolyK[11], SH);
    const int64_t k = (int32_t)(uint32_t)bits(kd);
    kd -= SH;
    double r = fma_(-kd, kExpPolyK[12], x);
    r = fma_(-kd, kExpPolyK[13], r);
    double p = fma_(r, kExpPolyK[0], kExpPolyK[1]);
#pragma unroll
    for (int i = 2; i < 11; ++i) p = fma_(r, p, kExpPolyK[i]);
    p = fma_(r, p, 0.5);
    p = fma_(r * r, p, r);  // exp(r) - 1
    const double m = 1.0 + p;
    const double res = from_bits(bits(m) + ((uint64_t)k << 52));
    return x < -708.0 ? 0.0 : res;  // NaN passes (the comparison is false)
}

// sum_k log(v_k) as one log of a running product: the product's exponent is
// peeled off after every factor (integer ops), so the mantissa m stays in [1, 2).
// Factors outside [2^-999, 2^1000) (subnormal, zero, huge, non-finite, negative)
// take their own libm-class log instead, so the product is never subnormal and
// never rounds more than a normal multiply does.
struct LogProd {
    double m = 1.0, acc = 0.0;
    int64_t ex = 0;
    SMC_HDM void add(double v)
    {
        const uint64_t ev = bits(v) >> 52;  // biased exponent (sign bit -> >= 2048)
        if (ev - 24u >= 2000u) {
            acc += smc_fm::log(v);
            return;
        }
        m *= v;  // in [2^-999, 2^1001): normal
        const uint64_t b = bits(m);
        ex += (int64_t)(b >> 52) - 1023;
        m = from_bits((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
    }
    SMC_HDM double result() const
    {
        const double e = (double)ex;  // e LN2_HI is exact for |e| < 2^11, rounded once beyond
        return acc + (e * 0x1.62e42fefa3800p-1 + (smc_fm::log(m) + e * 0x1.ef35793c76730p-45));
    }
};

}  // namespace smc_fm
