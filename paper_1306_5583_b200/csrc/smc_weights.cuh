// smc_weights.cuh -- the one-pass log-sum-exp / ESS reduction shared by the
// WeightSet kernels and the fused PF move kernel.
#pragma once
#include "smc_common.cuh"

namespace smc {

// Per-block partial of the normalization pass: block max of the raw log
// weights and sum_i e_i, sum_i e_i^2 with e_i = exp(v_i - bmax).
struct LsePartial {
    double m, s1, s2;
};

// Block-wide partial for ONE value per thread (v = -inf for idle threads).
// Block max first, then a single exp per element (no online rescaling).
template <int NT>
SMC_DEV LsePartial block_lse_partial(double v)
{
    __shared__ double sm_m[NT / 32];
    __shared__ double sm_s1[NT / 32], sm_s2[NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double m = warp_max(v);
    if (lane == 0) sm_m[warp] = m;
    __syncthreads();
    double bm = sm_m[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) bm = fmax(bm, sm_m[w]);
    // table exp (smc_fastmath.h, <= 0.52 ulp; -inf -> 0) from the L1-resident global table
    double e = smc_fm::exp(v - bm, smc_fm::kExpTab);
    double s1 = warp_sum(e), s2 = warp_sum(e * e);
    if (lane == 0) { sm_s1[warp] = s1; sm_s2[warp] = s2; }
    __syncthreads();
    LsePartial p{bm, 0.0, 0.0};
    if (threadIdx.x == 0) {
        for (int w = 0; w < NT / 32; ++w) { p.s1 += sm_s1[w]; p.s2 += sm_s2[w]; }
    }
    return p;  // valid in thread 0
}

// Combine two partials (either may be empty: m = -inf).
SMC_DEV LsePartial lse_combine(LsePartial a, LsePartial b)
{
    if (a.m == -INFINITY) return b;
    if (b.m == -INFINITY) return a;
    if (a.m >= b.m) {
        const double f = exp(b.m - a.m);
        return LsePartial{a.m, a.s1 + b.s1 * f, a.s2 + b.s2 * (f * f)};
    }
    const double f = exp(a.m - b.m);
    return LsePartial{b.m, b.s1 + a.s1 * f, b.s2 + a.s2 * (f * f)};
}

}  // namespace smc

// Finalize over block partials (one block, fixed combine order => deterministic).
// mode: SMC_W_* of the update (ADD_LOG sets nc_inc and optionally log_zconst).
// `scratch` needs smc_lse_scratch_bytes() bytes of device memory.
size_t smc_lse_scratch_bytes();
void smc_launch_lse_finalize(const smc::LsePartial *parts, int nparts, smc_wstate *st, int64_t n, int mode,
                             int accumulate_nc, cudaStream_t s, void *scratch, const double2 *mon_parts = nullptr,
                             double *mon_out = nullptr, double *partial_out = nullptr);
