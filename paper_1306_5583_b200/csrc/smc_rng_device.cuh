// smc_rng_device.cuh -- the reference's Philox4x32-10 streams on the device
// (rng.py:48-117): counter-based, so draw k of stream i is a pure function of
// (seed, i, k).  Self-contained and NVRTC-safe: included by the library's
// kernels (smc_common.cuh) and by user particle kernels compiled at run time
// (smc_user.cuh), so both draw bit-identical numbers.
#pragma once

#include "smc_fastmath.h"

#ifndef SMC_DEV
#define SMC_DEV __device__ __forceinline__
#endif

namespace smc {

// ---------------------------------------------------------------------------
// Philox4x32-10 (rng.py:48-72).  Counter = (draw_lo, draw_hi, stream_lo,
// stream_hi), key = (seed_lo, seed_hi); ten rounds, key bumped after each.
// ---------------------------------------------------------------------------
constexpr uint32_t PHILOX_M0 = 0xD2511F53u;
constexpr uint32_t PHILOX_M1 = 0xCD9E8D57u;
constexpr uint32_t PHILOX_W0 = 0x9E3779B9u;
constexpr uint32_t PHILOX_W1 = 0xBB67AE85u;

struct Key {
    uint32_t k0, k1;
    SMC_DEV uint32_t r0(int r) const { return k0 + (uint32_t)r * PHILOX_W0; }
    SMC_DEV uint32_t r1(int r) const { return k1 + (uint32_t)r * PHILOX_W1; }
};

// The ten round keys precomputed on the host.  Passed BY VALUE as a kernel
// parameter it lives in the constant bank, so each round's xor takes its key
// as a c[][] operand: no key-schedule instructions in the particle loop.
struct KeySched {
    uint32_t k0[10], k1[10];
    SMC_DEV uint32_t r0(int r) const { return k0[r]; }
    SMC_DEV uint32_t r1(int r) const { return k1[r]; }
};

SMC_DEV Key make_key(uint64_t seed) { return Key{(uint32_t)seed, (uint32_t)(seed >> 32)}; }

#ifndef __CUDACC_RTC__
inline KeySched make_key_sched(uint64_t seed)
{
    KeySched ks;
    for (int r = 0; r < 10; ++r) {
        ks.k0[r] = (uint32_t)seed + (uint32_t)r * PHILOX_W0;
        ks.k1[r] = (uint32_t)(seed >> 32) + (uint32_t)r * PHILOX_W1;
    }
    return ks;
}
#endif

template <class K>
SMC_DEV uint4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const K &key)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(PHILOX_M0, c0), lo0 = PHILOX_M0 * c0;
        const uint32_t hi1 = __umulhi(PHILOX_M1, c2), lo1 = PHILOX_M1 * c2;
        const uint32_t n0 = hi1 ^ c1 ^ key.r0(r);
        const uint32_t n2 = hi0 ^ c3 ^ key.r1(r);
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// 53-bit integer of draw `ctr` of stream `stream` (rng.py:81-82):
// ((w0 >> 5) << 26) | (w1 >> 6); the uniform is this times 2^-53, exactly.
template <int R0, class K>
SMC_DEV uint4 philox_rounds(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const K &key);

template <class K>
SMC_DEV uint64_t draw53(uint64_t ctr, uint64_t stream, const K &key)
{
    // the ten rounds with one mul.wide per product (philox_rounds): same bits as philox10
    const uint4 w = philox_rounds<0>((uint32_t)ctr, (uint32_t)(ctr >> 32), (uint32_t)stream,
                                     (uint32_t)(stream >> 32), key);
    return ((uint64_t)(w.x >> 5) << 26) | (uint64_t)(w.y >> 6);
}

template <class K>
SMC_DEV double u01_at(uint64_t ctr, uint64_t stream, const K &key)
{
    return __dmul_rn(__ull2double_rn(draw53(ctr, stream, key)), 1.0 / 9007199254740992.0);
}

// rng.py:85-91: Box-Muller cosine branch on 1 - u1, exactly two draws, from the
// two 53-bit draw integers.  (All TUs build with --fmad=false, so no contraction
// changes the rounding.)  Branch-free: log is smc_fastmath.h's table log (<= 0.55
// ulp, 99.6 % bit-identical to glibc), the radius root is sqrt_bm (bit-identical to
// IEEE sqrt on these inputs) and cos is cos_bm (<= 1.33 ulp, 83 % bit-identical to
// glibc, never more than 1 ulp away from it): the whole normal is one basic block.
// the fast-math tables a kernel staged in shared memory (null: the global tables)
struct FmTabs {
    const smc_fm::LogEntry *log = nullptr;
    const smc_fm::CosPoly *cos = nullptr;
};

// Box-Muller's two arguments from the draw integers: 1 - u1 = 1 - m1 2^-53 in [2^-53, 1]
// (exact, one FMA): a positive normal double, as log_core requires; fl(2 pi u2) =
// fl((2 pi 2^-53) m2), the power-of-two scale being exact
SMC_DEV double2 box_muller_args(uint64_t m1, uint64_t m2)
{
    return make_double2(__fma_rn(-__ull2double_rn(m1), 1.0 / 9007199254740992.0, 1.0),
                        __dmul_rn(__ull2double_rn(m2), (2.0 * 3.141592653589793) / 9007199254740992.0));
}
SMC_DEV double box_muller_from(double2 a, FmTabs tabs = FmTabs{})
{
    return smc_fm::sqrt_bm(-2.0 * smc_fm::log_core(a.x, tabs.log)) * smc_fm::cos_bm(a.y, tabs.cos);
}
SMC_DEV double box_muller53(uint64_t m1, uint64_t m2, FmTabs tabs = FmTabs{})
{
    return box_muller_from(box_muller_args(m1, m2), tabs);
}

template <class K>
SMC_DEV double normal_at(uint64_t ctr, uint64_t stream, const K &key)
{
    return box_muller53(draw53(ctr, stream, key), draw53(ctr + 1, stream, key));
}

// NZ consecutive normals of one stream (draws ctr .. ctr + 2 NZ - 1): every Philox
// block first (2 NZ independent integer chains the scheduler interleaves), then the
// NZ Box-Muller transforms.  Bit-identical to NZ calls of normal_at.
template <int NZ, class K>
SMC_DEV void normals_at(uint64_t ctr, uint64_t stream, const K &key, double (&z)[NZ], FmTabs tabs = FmTabs{})
{
    uint64_t m[2 * NZ];
#pragma unroll
    for (int j = 0; j < 2 * NZ; ++j) m[j] = draw53(ctr + (uint64_t)j, stream, key);
#pragma unroll
    for (int j = 0; j < NZ; ++j) z[j] = box_muller53(m[2 * j], m[2 * j + 1], tabs);
}

// Rounds R0..9 of philox10 (R0 = 0: the whole block).
// one 32x32 -> 64 product as a single mul.wide (ptxas otherwise may split it into a
// separate high and low multiply: two issue slots instead of one)
SMC_DEV void mulwide(uint32_t a, uint32_t m, uint32_t &hi, uint32_t &lo)
{
    asm("{\n\t.reg .u64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%1, %0}, p;\n\t}"
        : "=r"(hi), "=r"(lo) : "r"(a), "r"(m));
}

template <int R0, class K>
SMC_DEV uint4 philox_rounds(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const K &key)
{
#pragma unroll
    for (int r = R0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulwide(c0, PHILOX_M0, hi0, lo0);
        mulwide(c2, PHILOX_M1, hi1, lo1);
        const uint32_t n0 = hi1 ^ c1 ^ key.r0(r);
        const uint32_t n2 = hi0 ^ c3 ^ key.r1(r);
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// Every stream at the same draw count ctr with no carry into its high word over the next
// 16 draws (lo32(ctr) <= 2^32 - 16), and every stream index below 2^32 (the host checks
// both).  Then the round-1 M0 product of draw j, M0 * (lo32(ctr) + j), is the same for every
// stream, and so is round 2's M1 operand (hi of that product ^ round-1 key, the stream's high
// word being 0): both products come precomputed from the host (kernel-parameter, i.e.
// constant-bank, operands).  Per stream, round 1's M1 product and round 2's M0 product are
// common to all of its draws: each draw costs the 16 multiplies of rounds 3-10 instead of 20.
struct UniformCtr {
    uint32_t c1k;      // hi32(ctr) ^ round-1 key word 0
    uint32_t a[16];    // round 2: umulhi(M1, n2_j) ^ round-2 key word 0, n2_j = umulhi(M0, c0_j) ^ round-1 key word 1
    uint32_t b[16];    // round 2: M1 * n2_j (the next c1)
    uint32_t c[16];    // M0 * c0_j (round 1's next c3) ^ round-2 key word 1
};

#ifndef __CUDACC_RTC__
inline UniformCtr make_uniform_ctr(uint64_t ctr, const KeySched &ks)
{
    UniformCtr u;
    u.c1k = (uint32_t)(ctr >> 32) ^ ks.k0[0];
    for (int j = 0; j < 16; ++j) {
        const uint64_t p0 = (uint64_t)PHILOX_M0 * (uint32_t)((uint32_t)ctr + (uint32_t)j);
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ ks.k1[0];  // round 1 with stream hi word 0
        const uint64_t p1 = (uint64_t)PHILOX_M1 * n2;            // round 2's M1 product
        u.a[j] = (uint32_t)(p1 >> 32) ^ ks.k0[1];
        u.b[j] = (uint32_t)p1;
        u.c[j] = (uint32_t)p0 ^ ks.k1[1];
    }
    return u;
}
#endif

// The 53-bit draw integers of draws ctr .. ctr + ND - 1 of one stream, for the counter `u`
// describes and stream < 2^32 (bit-identical to draw53).
template <int ND, class K>
SMC_DEV void draws_uniform(const UniformCtr &u, uint64_t stream, const K &key, uint64_t (&m)[ND])
{
    static_assert(ND <= 16, "UniformCtr holds 16 draws");
    const uint32_t c2 = (uint32_t)stream;
    const uint32_t hi1 = __umulhi(PHILOX_M1, c2), lo1 = PHILOX_M1 * c2;  // round 1, every draw
    const uint32_t n0 = hi1 ^ u.c1k;
    const uint32_t hi0b = __umulhi(PHILOX_M0, n0), lo0b = PHILOX_M0 * n0;  // round 2, every draw
#pragma unroll
    for (int j = 0; j < ND; ++j) {
        const uint4 w = philox_rounds<2>(u.a[j] ^ lo1, u.b[j], hi0b ^ u.c[j], lo0b, key);
        m[j] = ((uint64_t)(w.x >> 5) << 26) | (uint64_t)(w.y >> 6);
    }
}

// normals_at(ctr, stream, ...) for the counter `u` describes and stream < 2^32: bit-identical.
template <int NZ, class K>
SMC_DEV void normals_uniform(const UniformCtr &u, uint64_t stream, const K &key, double (&z)[NZ],
                             FmTabs tabs = FmTabs{})
{
    uint64_t m[2 * NZ];
    draws_uniform<2 * NZ>(u, stream, key, m);
#pragma unroll
    for (int j = 0; j < NZ; ++j) z[j] = box_muller53(m[2 * j], m[2 * j + 1], tabs);
}

// rng.py:94-117: Marsaglia-Tsang (+ boost below shape 1); advances *ctr by the
// variable number of draws it consumes.
template <class K>
SMC_DEV double gamma_from(uint64_t &ctr, uint64_t stream, const K &key, double shape)
{
    double boost = 1.0;
    double a = shape;
    if (a < 1.0) {
        const double u = 1.0 - u01_at(ctr, stream, key);
        ctr += 1;
        boost = pow(u, 1.0 / a);
        a = a + 1.0;
    }
    const double d = a - 1.0 / 3.0;
    const double c = 1.0 / sqrt(9.0 * d);
    for (;;) {
        const double x = normal_at(ctr, stream, key);
        ctr += 2;
        const double t = 1.0 + c * x;
        if (t <= 0.0) continue;
        const double v = t * t * t;
        const double u = 1.0 - u01_at(ctr, stream, key);
        ctr += 1;
        if (smc_fm::log(u) < 0.5 * x * x + d - d * v + d * smc_fm::log(v)) return boost * d * v;
    }
}

}  // namespace smc
