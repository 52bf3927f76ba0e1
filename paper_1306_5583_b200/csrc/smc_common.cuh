// smc_common.cuh -- device building blocks shared by every sm_100a kernel of the
// SMC hot path: the reference's Philox4x32-10 stream (rng.py:48-117), exact
// 128-bit helpers for the integer resampling contract, warp/block scans and
// the stream-status plumbing of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/smc_abi.h"
#include "smc_rng_device.cuh"

typedef unsigned __int128 u128;

// Programmatic dependent launch (sm_90+): kernels of the hot chain are launched with
// the programmatic-stream-serialization attribute, so a kernel's launch and block
// rasterization overlap the previous kernel's tail; every such kernel starts with
// SMC_PDL_WAIT (griddepcontrol.wait: all prerequisite grids complete and their memory
// visible), so stream-order semantics are unchanged.  Without the attribute the wait
// returns at once.
#define SMC_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
// ... and a kernel may let its dependent launch before it finishes (the dependent still waits in
// SMC_PDL_WAIT for this grid's completion and memory): used after a block's main loop, so the
// next kernel's blocks get rasterized while the last wave finishes its reductions
#ifndef SMC_NO_PDL_TRIGGER
#define SMC_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#else
#define SMC_PDL_TRIGGER() do { } while (0)
#endif

// Every kernel launch of the library bumps this counter (smc_launch_count in the ABI): the bench
// reports how many of OUR kernels ran in its timed region from it, not from a guess.
#include <atomic>
inline std::atomic<unsigned long long> &smc_launch_counter()
{
    static std::atomic<unsigned long long> c{0};
    return c;
}
#define SMC_COUNT_LAUNCH() smc_launch_counter().fetch_add(1, std::memory_order_relaxed)

// Checked build (-DSMC_CHECKED=1; tools/gpu/checked.sh): SMC_CHECK(cond) guards the shared- and
// global-memory indices the kernels compute (staging slices, rank tables, bins, sub-buckets,
// parent indices).  A violated check is counted, never trapped (the GPU stays healthy and the
// test that caused it keeps running): every translation unit keeps its own device counters and
// registers a reader, and smc_check_failures() (ABI) sums them and names the first failing line.
// The stand-in for compute-sanitizer's memcheck on a pool where the sanitizer is closed.
#if SMC_CHECKED
static __device__ unsigned long long smc_chk_fail_d, smc_chk_line_d;
#define SMC_CHECK(c)                                                                   \
    do {                                                                               \
        if (!(c)) {                                                                    \
            atomicAdd(&smc_chk_fail_d, 1ull);                                          \
            atomicCAS(&smc_chk_line_d, 0ull, (unsigned long long)__LINE__);            \
        }                                                                              \
    } while (0)
#else
#define SMC_CHECK(c) do { } while (0)
#endif
typedef void (*smc_chk_reader)(uint64_t *fails, uint64_t *line, const char **file);
#include <vector>
inline std::vector<smc_chk_reader> &smc_chk_readers()
{
    static std::vector<smc_chk_reader> v;
    return v;
}
#if SMC_CHECKED
static void smc_chk_read_tu(uint64_t *fails, uint64_t *line, const char **file)
{
    unsigned long long f = 0, l = 0;
    cudaMemcpyFromSymbol(&f, smc_chk_fail_d, sizeof f);
    cudaMemcpyFromSymbol(&l, smc_chk_line_d, sizeof l);
    *fails += f;
    if (l && !*line) {
        *line = l;
        *file = __BASE_FILE__;
    }
}
static const bool smc_chk_registered = (smc_chk_readers().push_back(&smc_chk_read_tu), true);
#endif

template <typename... KArgs, typename... Args>
inline void smc_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    SMC_COUNT_LAUNCH();
}

namespace smc {

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

// ... and the first (lowest-index) failing particle: a status word is
// followed, 8 bytes on, by its record of the first failing index, stored as INT32_MAX - index
// so that an atomicMax keeps the lowest index and 0 means "none" (smc_abi.h, smc_status).
SMC_DEV void raise_status_at(int32_t *status, int32_t code, int64_t index)
{
    if (!status) return;
    atomicCAS(reinterpret_cast<int *>(status), 0, code);
    if (index >= 0 && index < 0x7fffffff) atomicMax(reinterpret_cast<int *>(status + 2), 0x7fffffff - (int)index);
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

// Full, 32-byte-aligned tiles skip the transpose: each thread's ITEMS
// consecutive items are whole 32-byte sectors, read / written with 256-bit
// accesses (every sector of every instruction fully used).  Partial tiles take
// the shared-memory path.  The choice is per block (uniform), so the barriers
// of the fallback stay convergent.
SMC_DEV void ld_sector(const void *p, uint64_t (&w)[4])
{
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p));
}
SMC_DEV void st_sector(void *p, const uint64_t (&w)[4])
{
    asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(w[0]), "l"(w[1]), "l"(w[2]), "l"(w[3])
                 : "memory");
}

// 64-bit words <-> items (bit casts for double, value casts for the integer types)
template <typename T>
SMC_DEV T from_u64(uint64_t w) { return (T)w; }
template <>
SMC_DEV double from_u64<double>(uint64_t w) { return __longlong_as_double((long long)w); }
template <typename T>
SMC_DEV uint64_t to_u64(T v) { return (uint64_t)v; }
template <>
SMC_DEV uint64_t to_u64<double>(double v) { return (uint64_t)__double_as_longlong(v); }

template <int NT, int ITEMS, typename T>
SMC_DEV bool vector_tile(const T *g, int64_t base, int64_t n)
{
    return (ITEMS * sizeof(T)) % 32 == 0 && (sizeof(T) == 4 || sizeof(T) == 8) && base + NT * ITEMS <= n &&
           (((uintptr_t)(g + base)) & 31) == 0;
}

template <int NT, int ITEMS, typename T>
SMC_DEV void load_blocked(const T *__restrict__ g, int64_t base, int64_t n, T (&v)[ITEMS], T *sm, T pad)
{
    if (vector_tile<NT, ITEMS, T>(g, base, n)) {
        const char *p = (const char *)(g + base + (int64_t)threadIdx.x * ITEMS);
#pragma unroll
        for (int c = 0; c < (int)(ITEMS * sizeof(T)) / 32; ++c) {
            uint64_t w[4];
            ld_sector(p + 32 * c, w);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (sizeof(T) == 8) {
                    v[c * 4 + k] = from_u64<T>(w[k]);
                } else {
                    v[c * 8 + 2 * k] = (T)(uint32_t)w[k];
                    v[c * 8 + 2 * k + 1] = (T)(uint32_t)(w[k] >> 32);
                }
            }
        }
        return;
    }
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
    if (vector_tile<NT, ITEMS, T>(g, base, n)) {
        char *p = (char *)(g + base + (int64_t)threadIdx.x * ITEMS);
#pragma unroll
        for (int c = 0; c < (int)(ITEMS * sizeof(T)) / 32; ++c) {
            uint64_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (sizeof(T) == 8)
                    w[k] = to_u64<T>(v[c * 4 + k]);
                else
                    w[k] = (uint64_t)(uint32_t)v[c * 8 + 2 * k] | ((uint64_t)(uint32_t)v[c * 8 + 2 * k + 1] << 32);
            }
            st_sector(p + 32 * c, w);
        }
        return;
    }
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
