// smc_rng.cu -- device Philox streams (replaces pkg/src/smckit/rng.py).
//
// Uniforms are bit-identical to the reference (integer construction, rng.py:81-82).
// Normals/gammas use libdevice log/cos/sqrt/pow and agree with glibc to a few ulp.
#include "smc_common.cuh"

using namespace smc;

__global__ void k_philox_blocks(const uint4 *__restrict__ ctr, int64_t n, Key key, uint4 *__restrict__ out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 c = ctr[i];
    out[i] = philox10(c.x, c.y, c.z, c.w, key);
}

// fill_u01 / fill_std_normal (rng.py:120-131): draw k of one stream uses
// counter c0+k (u01) or c0+2k, c0+2k+1 (normal) -- independent, so parallel.
__global__ void k_fill_parallel(int kind, Key key, uint64_t stream, const uint64_t *__restrict__ ctr,
                                double mean, double scale, double *__restrict__ out, int64_t n)
{
    const uint64_t c0 = *ctr;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        if (kind == SMC_DRAW_U01) out[k] = u01_at(c0 + (uint64_t)k, stream, key);
        else out[k] = mean + scale * normal_at(c0 + 2 * (uint64_t)k, stream, key);
    }
}

__global__ void k_advance(uint64_t *ctr, uint64_t by) { *ctr += by; }

// fill_std_gamma (rng.py:132-135): data-dependent draw count => one thread.
__global__ void k_fill_gamma(Key key, uint64_t stream, uint64_t *ctr, double shape, double scale,
                             double *__restrict__ out, int64_t n)
{
    uint64_t c = *ctr;
    for (int64_t k = 0; k < n; ++k) out[k] = scale * gamma_from(c, stream, key, shape);
    *ctr = c;
}

// One draw per stream (rng.py:75-117 per particle).
__global__ void k_draw_streams(int kind, Key key, uint64_t first, int64_t n, uint64_t *__restrict__ ctrs,
                               double shape, double mean, double scale, double *__restrict__ out)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint64_t s = first + (uint64_t)j;
    uint64_t c = ctrs[s];
    double v;
    if (kind == SMC_DRAW_U01) { v = u01_at(c, s, key); c += 1; }
    else if (kind == SMC_DRAW_NORMAL) { v = mean + scale * normal_at(c, s, key); c += 2; }
    else { v = scale * gamma_from(c, s, key, shape); }
    ctrs[s] = c;
    out[j] = v;
}

static inline int grid_for(int64_t n, int bs, int cap = 148 * 64)
{
    int64_t g = (n + bs - 1) / bs;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

extern "C" int smc_philox_blocks(const uint32_t *ctr4, int64_t n, uint64_t seed, uint32_t *out4, void *stream)
{
    if (n < 0 || (n && (!ctr4 || !out4))) return smc_set_error(SMC_EINVAL, "smc_philox_blocks: bad args");
    if (!n) return SMC_OK;
    const int bs = 256;
    k_philox_blocks<<<(unsigned)((n + bs - 1) / bs), bs, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const uint4 *>(ctr4), n, Key{(uint32_t)seed, (uint32_t)(seed >> 32)},
        reinterpret_cast<uint4 *>(out4));
    SMC_COUNT_LAUNCH();
    return smc_check_launch("smc_philox_blocks");
}

extern "C" int smc_rng_fill(int kind, uint64_t seed, uint64_t stream_index, uint64_t *ctrs, double shape,
                            double mean, double scale, double *out, int64_t n, void *stream)
{
    if (n < 0 || !ctrs || (n && !out) || kind < 0 || kind > 2)
        return smc_set_error(SMC_EINVAL, "smc_rng_fill: bad args");
    if (kind == SMC_DRAW_NORMAL && !(scale > 0.0))
        return smc_set_error(SMC_EINVAL, "normal needs sd > 0, got sd=%g", scale);  // rng.py:198
    if (kind == SMC_DRAW_GAMMA && !(shape > 0.0 && scale > 0.0))
        return smc_set_error(SMC_EINVAL, "gamma needs shape > 0 and scale > 0");  // rng.py:209
    if (!n) return SMC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const Key key{(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint64_t *ctr = ctrs + stream_index;
    if (kind == SMC_DRAW_GAMMA) {
        k_fill_gamma<<<1, 1, 0, s>>>(key, stream_index, ctr, shape, scale, out, n);
        SMC_COUNT_LAUNCH();
    } else {
        const int bs = 256;
        k_fill_parallel<<<grid_for(n, bs), bs, 0, s>>>(kind, key, stream_index, ctr, mean, scale, out, n);
        k_advance<<<1, 1, 0, s>>>(ctr, (uint64_t)n * (kind == SMC_DRAW_U01 ? 1u : 2u));
        SMC_COUNT_LAUNCH();
        SMC_COUNT_LAUNCH();
    }
    return smc_check_launch("smc_rng_fill");
}

extern "C" int smc_rng_draw_streams(int kind, uint64_t seed, uint64_t first_stream, int64_t n, uint64_t *ctrs,
                                    double shape, double mean, double scale, double *out, void *stream)
{
    if (n < 0 || (n && (!ctrs || !out)) || kind < 0 || kind > 2)
        return smc_set_error(SMC_EINVAL, "smc_rng_draw_streams: bad args");
    if (kind == SMC_DRAW_NORMAL && !(scale > 0.0)) return smc_set_error(SMC_EINVAL, "normal needs sd > 0");
    if (kind == SMC_DRAW_GAMMA && !(shape > 0.0 && scale > 0.0))
        return smc_set_error(SMC_EINVAL, "gamma needs shape > 0 and scale > 0");
    if (!n) return SMC_OK;
    const int bs = 256;
    k_draw_streams<<<(unsigned)((n + bs - 1) / bs), bs, 0, (cudaStream_t)stream>>>(
        kind, Key{(uint32_t)seed, (uint32_t)(seed >> 32)}, first_stream, n, ctrs, shape, mean, scale, out);
    SMC_COUNT_LAUNCH();
    return smc_check_launch("smc_rng_draw_streams");
}
