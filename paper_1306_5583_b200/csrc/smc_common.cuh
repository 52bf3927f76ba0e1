// smc_common.cuh -- device building blocks shared by every sm_100a kernel of the
// SMC hot path: the reference's Philox4x32-10 stream (rng.py:48-117), exact
// 128-bit helpers for the integer resampling contract, warp/block scans and
// the stream-status plumbing of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/smc_abi.h"
#include "smc_fastmath.h"

typedef unsigned __int128 u128;

#define SMC_DEV __device__ __forceinline__

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
};

SMC_DEV Key make_key(uint64_t seed) { return Key{(uint32_t)seed, (uint32_t)(seed >> 32)}; }

SMC_DEV uint4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, Key key)
{
    uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(PHILOX_M0, c0), lo0 = PHILOX_M0 * c0;
        const uint32_t hi1 = __umulhi(PHILOX_M1, c2), lo1 = PHILOX_M1 * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += PHILOX_W0;
        k1 += PHILOX_W1;
    }
    return make_uint4(c0, c1, c2, c3);
}

// 53-bit integer of draw `ctr` of stream `stream` (rng.py:81-82):
// ((w0 >> 5) << 26) | (w1 >> 6); the uniform is this times 2^-53, exactly.
SMC_DEV uint64_t draw53(uint64_t ctr, uint64_t stream, Key key)
{
    const uint4 w = philox10((uint32_t)ctr, (uint32_t)(ctr >> 32), (uint32_t)stream,
                             (uint32_t)(stream >> 32), key);
    return ((uint64_t)(w.x >> 5) << 26) | (uint64_t)(w.y >> 6);
}

SMC_DEV double u01_at(uint64_t ctr, uint64_t stream, Key key)
{
    return __dmul_rn(__ull2double_rn(draw53(ctr, stream, key)), 1.0 / 9007199254740992.0);
}

// rng.py:85-91: Box-Muller cosine branch on 1 - u1, exactly two draws.
// (All TUs build with --fmad=false, so no contraction changes the rounding;
// log is smc_fastmath.h's table log (<= 0.55 ulp, 99.6 % bit-identical to glibc,
// 8 % cheaper than libdevice on B200); cos is libdevice's (the fdlibm-style
// smc_fm::cos diverges per quadrant and measured 40 % slower); sqrt is IEEE.)
SMC_DEV double normal_at(uint64_t ctr, uint64_t stream, Key key)
{
    const double u1 = u01_at(ctr, stream, key);
    const double u2 = u01_at(ctr + 1, stream, key);
    return sqrt(-2.0 * smc_fm::log(1.0 - u1)) * cos((2.0 * 3.141592653589793) * u2);
}

// rng.py:94-117: Marsaglia-Tsang (+ boost below shape 1); advances *ctr by the
// variable number of draws it consumes.
SMC_DEV double gamma_from(uint64_t &ctr, uint64_t stream, Key key, double shape)
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

// ---------------------------------------------------------------------------
// Normalized log-weights from the raw vector + device record (smc_abi.h).
// ---------------------------------------------------------------------------
struct NormLw {
    double m, ls;
    bool eq;
    double weq;  // the equal weight 1/N (valid when eq)
    SMC_DEV double operator()(double raw) const { return eq ? -ls : (raw - m) - ls; }
    SMC_DEV bool needs_raw() const { return !eq; }
};
SMC_DEV NormLw norm_of(const smc_wstate *st)
{
    return NormLw{st->max_raw, st->log_sum, st->equal != 0, st->w_equal};
}

// ---------------------------------------------------------------------------
// Device status: first error wins ("first failing ... reported").
// ---------------------------------------------------------------------------
SMC_DEV void raise_status(int32_t *status, int32_t code)
{
    if (status) atomicCAS(reinterpret_cast<int *>(status), 0, code);
}

// ---------------------------------------------------------------------------
// Warp / block scans and reductions.
// ---------------------------------------------------------------------------
template <typename T>
SMC_DEV T warp_inclusive_sum(T v)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

template <typename T>
SMC_DEV T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

SMC_DEV double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Exclusive block scan of T over NT threads; returns the exclusive prefix of
// this thread and writes the block total to *total.  `sm` needs NT/32 + 1 slots.
template <int NT, typename T>
SMC_DEV T block_exclusive_sum(T v, T *sm, T *total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    T inc = warp_inclusive_sum(v);
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? sm[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < NW) sm[lane] = wi - w;
        if (lane == NW - 1) sm[NW] = wi;
    }
    __syncthreads();
    T ex = sm[warp] + inc - v;
    *total = sm[NW];
    __syncthreads();
    return ex;
}

// Coalesced tile I/O.  Lanes of a warp touch contiguous addresses (one 128-byte
// line per 32 x 4 B); the tile is transposed through shared memory so each
// thread owns ITEMS consecutive items ("blocked" order, what scans need).  One
// pad word per 128 B of shared memory keeps both phases bank-conflict free.
template <typename T>
SMC_DEV int tpad(int i) { return i + i / (128 / (int)sizeof(T)); }
template <typename T, int NT, int ITEMS>
constexpr int tile_smem_elems() { return NT * ITEMS + NT * ITEMS / (128 / (int)sizeof(T)) + 1; }

template <int NT, int ITEMS, typename T>
SMC_DEV void load_blocked(const T *__restrict__ g, int64_t base, int64_t n, T (&v)[ITEMS], T *sm, T pad)
{
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const int li = j * NT + threadIdx.x;
        sm[tpad<T>(li)] = base + li < n ? g[base + li] : pad;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) v[j] = sm[tpad<T>(threadIdx.x * ITEMS + j)];
    __syncthreads();
}

template <int NT, int ITEMS, typename T>
SMC_DEV void store_blocked(T *__restrict__ g, int64_t base, int64_t n, const T (&v)[ITEMS], T *sm)
{
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) sm[tpad<T>(threadIdx.x * ITEMS + j)] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const int li = j * NT + threadIdx.x;
        if (base + li < n) g[base + li] = sm[tpad<T>(li)];
    }
    __syncthreads();
}

// u128 has no shuffle; split in halves.
SMC_DEV u128 shfl_xor_u128(u128 v, int o)
{
    uint64_t lo = (uint64_t)v, hi = (uint64_t)(v >> 64);
    lo = __shfl_xor_sync(0xffffffffu, lo, o);
    hi = __shfl_xor_sync(0xffffffffu, hi, o);
    return ((u128)hi << 64) | lo;
}

// floor(a*b / d) for the stratum search, exact: fp64 estimate + integer fix-up.
SMC_DEV uint64_t div_floor_u128(u128 num, uint64_t d)
{
    double est = (double)num / (double)d;
    uint64_t s = est <= 0.0 ? 0 : (uint64_t)est;
    // fix-up: the estimate is within a couple of units of the truth
    while ((u128)s * d > num) --s;
    while ((u128)(s + 1) * d <= num) ++s;
    return s;
}

}  // namespace smc

// Launch-error plumbing for the ABI layer.
int smc_set_error(int code, const char *fmt, ...);
int smc_check_launch(const char *what);
