// smc_weights.cu -- WeightSet on the device (replaces smckit.weights),
// the ESS trigger and the monitor/path weighted sums
// (SPEC.md:320-333, :403-416).
//
// Storage: lw_raw[N] plus a device smc_wstate {max_raw, log_sum, ess, ...}.  The
// normalized log-weight is (lw_raw - max_raw) - log_sum (or -log N after
// set_equal_weight, which only flips a flag) so normalization never needs a
// second write pass.
#include "smc_weights.cuh"

using namespace smc;

namespace {

constexpr int WB = 256;  // threads per block of the per-element passes

// One element per thread: new raw log-weight for the requested mutation.
__global__ void __launch_bounds__(WB) k_weights_pass(int mode, double *__restrict__ lw_raw,
                                                      const double *__restrict__ values, int64_t n,
                                                      smc_wstate *st, LsePartial *__restrict__ parts)
{
    SMC_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * WB + threadIdx.x;
    double v = -INFINITY;
    if (i < n) {
        double prev = 0.0;
        if (mode == SMC_W_ADD_LOG || mode == SMC_W_MUL_LIN) {
            const NormLw nl = norm_of(st);
            prev = nl(nl.needs_raw() ? lw_raw[i] : 0.0);
        }
        const double x = values[i];
        switch (mode) {
        case SMC_W_SET_LOG: v = x; break;
        case SMC_W_ADD_LOG: v = prev + x; break;
        case SMC_W_SET_LIN: v = (x >= 0.0) ? log(x) : NAN; break;
        default: v = (x >= 0.0) ? prev + log(x) : NAN; break;  // MUL_LIN
        }
        if (isnan(v) || v == INFINITY) {
            raise_status_at(&st->status, SMC_ENORMALIZE, i);
            v = -INFINITY;
        }
        lw_raw[i] = v;
    }
    LsePartial p = block_lse_partial<WB>(v);
    if (threadIdx.x == 0) parts[blockIdx.x] = p;
}

constexpr int FB = 256;   // threads per finalize block
constexpr int FG = 148;   // level-1 finalize blocks (one per SM)

// Finalize = two small launches so the ~N/256 block partials are read by the
// whole GPU, not one SM: level 1 (FG blocks) reduces a contiguous slice each,
// level 2 (one block) combines the FG results in index order (deterministic).
// Each level is two-phase so every exp is independent: M = max m_b, then
// s1 = sum s1_b e^{m_b - M}, s2 = sum s2_b e^{2(m_b - M)}.  Optional monitor
// partials (mon_parts[b] = sum_i W_i h(X_i) over block b) ride along.
// CG: the partials were written by other blocks of the SAME grid (the last-block combine):
// loaded through L2 (ld.global.cg), never the non-coherent path.
template <bool CG>
SMC_DEV LsePartial ld_part(const LsePartial *p)
{
    if (CG) return LsePartial{__ldcg(&p->m), __ldcg(&p->s1), __ldcg(&p->s2)};
    return *p;
}
template <bool CG>
SMC_DEV double2 ld_mon(const double2 *p)
{
    if (CG) return __ldcg(p);
    return *p;
}
template <bool CG = false>
SMC_DEV void lse_slice(const LsePartial *parts, const double2 *mon, int b0, int b1, LsePartial *out, double2 *out_mon)
{
    __shared__ double sm_a[FB / 32], sm_b[FB / 32], sm_c[FB / 32], sm_d[FB / 32];
    __shared__ double s_M;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double m = -INFINITY;
    for (int b = b0 + threadIdx.x; b < b1; b += FB) m = fmax(m, ld_part<CG>(parts + b).m);
    m = warp_max(m);
    if (lane == 0) sm_a[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double M = sm_a[0];
        for (int w = 1; w < FB / 32; ++w) M = fmax(M, sm_a[w]);
        s_M = M;
    }
    __syncthreads();
    const double M = s_M;
    double s1 = 0.0, s2 = 0.0, h0 = 0.0, h1 = 0.0;
    for (int b = b0 + threadIdx.x; b < b1; b += FB) {
        const LsePartial p = ld_part<CG>(parts + b);
        if (p.m != -INFINITY) {
            const double f = exp(p.m - M);
            s1 += p.s1 * f;
            s2 += p.s2 * (f * f);
        }
        if (mon) {
            const double2 hm = ld_mon<CG>(mon + b);
            h0 += hm.x;
            h1 += hm.y;
        }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    h0 = warp_sum(h0);
    h1 = warp_sum(h1);
    __syncthreads();
    if (lane == 0) { sm_a[warp] = s1; sm_b[warp] = s2; sm_c[warp] = h0; sm_d[warp] = h1; }
    __syncthreads();
    if (threadIdx.x == 0) {
        LsePartial t{M, 0.0, 0.0};
        double H0 = 0.0, H1 = 0.0;
        for (int w = 0; w < FB / 32; ++w) { t.s1 += sm_a[w]; t.s2 += sm_b[w]; H0 += sm_c[w]; H1 += sm_d[w]; }
        *out = t;
        *out_mon = make_double2(H0, H1);
    }
}

// The state update shared by the single-GPU finalize and the multi-GPU combine.
SMC_DEV void apply_lse(smc_wstate *st, LsePartial t, int64_t n, int mode, int accumulate_nc)
{
    if (t.m == -INFINITY || !(t.s1 > 0.0)) {
        raise_status(&st->status, SMC_ENORMALIZE);  // SPEC.md:45 all -inf
        return;
    }
    const double ls = log(t.s1);
    const double lse = t.m + ls;
    st->lse = lse;
    st->max_raw = t.m;
    st->log_sum = ls;
    st->ess = (t.s1 * t.s1) / t.s2;  // 1 / sum W^2 with W = e / s1
    st->ess_over_n = st->ess / (double)n;
    st->equal = 0;
    if (mode == SMC_W_ADD_LOG) {
        // previous lw was normalized => log sum_i W_{t-1,i} exp(incw_i) = lse
        st->nc_inc = lse;
        if (accumulate_nc) st->log_zconst += lse;
    } else if (mode == SMC_W_SET_LOG && accumulate_nc) {
        // first weighting from the equal-weight prior sample: log (1/N) sum_i exp(v_i)
        st->nc_inc = lse - log((double)n);
        st->log_zconst = st->nc_inc;
    }
}

// One launch for both levels: FG blocks each combine a slice of the block partials; the last
// block to finish (a ticket in the weight record, reset by that block) combines the FG results
// in index order -- the same arithmetic as two launches, one launch gap less per weight update.
// partial_out != NULL (a shard of a multi-GPU system): export {max, sum e, sum e^2, monitor0,
// monitor1} instead of updating the state; the ranks then allgather and smc_weights_combine them
// in rank order.
__global__ void __launch_bounds__(FB) k_lse_reduce(const LsePartial *__restrict__ parts, int nparts,
                                                   const double2 *__restrict__ mon, LsePartial *l2, double2 *l2mon,
                                                   smc_wstate *st, int64_t n, int mode, int accumulate_nc,
                                                   double *mon_out, double *partial_out)
{
    SMC_PDL_WAIT();
    const int per = (nparts + FG - 1) / FG;
    const int b0 = min(nparts, (int)blockIdx.x * per), b1 = min(nparts, b0 + per);
    lse_slice(parts, mon, b0, b1, l2 + blockIdx.x, l2mon + blockIdx.x);
    __shared__ int s_last;
    if (threadIdx.x == 0) {  // this block's l2 entry (written by thread 0 above) before its ticket
        __threadfence();
        s_last = atomicAdd(&st->lse_ticket, 1u) == (unsigned)FG - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ LsePartial s_t;
    __shared__ double2 s_h;
    const bool has_mon = mon != nullptr;
    lse_slice<true>(l2, has_mon ? l2mon : nullptr, 0, FG, &s_t, &s_h);
    if (threadIdx.x == 0) {
        st->lse_ticket = 0;
        const LsePartial t = s_t;
        if (partial_out) {
            partial_out[0] = t.m;
            partial_out[1] = t.s1;
            partial_out[2] = t.s2;
            partial_out[3] = has_mon ? s_h.x : 0.0;
            partial_out[4] = has_mon ? s_h.y : 0.0;
            return;
        }
        if (has_mon && mon_out) { mon_out[0] = s_h.x; mon_out[1] = s_h.y; }
        apply_lse(st, t, n, mode, accumulate_nc);
    }
}

// Multi-GPU: combine G exported shard partials (stride SMC_PARTIAL_STRIDE) in
// rank order -- every rank computes bit-identical state (unlike an allreduce).
__global__ void k_lse_combine(const double *__restrict__ parts, int G, smc_wstate *st, int64_t n_total, int mode,
                              int accumulate_nc, double *mon_out)
{
    SMC_PDL_WAIT();
    double M = -INFINITY;
    for (int g = 0; g < G; ++g) M = fmax(M, parts[g * SMC_PARTIAL_STRIDE]);
    LsePartial t{M, 0.0, 0.0};
    double h0 = 0.0, h1 = 0.0;
    for (int g = 0; g < G; ++g) {
        const double *p = parts + g * SMC_PARTIAL_STRIDE;
        if (p[0] != -INFINITY) {
            const double f = exp(p[0] - M);
            t.s1 += p[1] * f;
            t.s2 += p[2] * (f * f);
        }
        h0 += p[3];
        h1 += p[4];
    }
    if (mon_out) { mon_out[0] = h0; mon_out[1] = h1; }
    apply_lse(st, t, n_total, mode, accumulate_nc);
}

__global__ void k_set_equal(smc_wstate *st, int64_t n, const int32_t *gate)
{
    SMC_PDL_WAIT();
    if (gate && *gate == 0) return;
    st->equal = 1;
    st->lse = log((double)n);  // consistent with lw_raw == 0 everywhere
    st->max_raw = 0.0;
    st->log_sum = log((double)n);
    st->w_equal = 1.0 / (double)n;
    st->ess = (double)n;
    st->ess_over_n = 1.0;
}

__global__ void k_weights_read(int what, const double *__restrict__ lw_raw, const smc_wstate *st, int64_t n,
                               double *__restrict__ out)
{
    SMC_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const NormLw nl = norm_of(st);
    const double l = nl(nl.needs_raw() ? lw_raw[i] : 0.0);
    // equal weights are exp(-log N): N is the GLOBAL count of a sharded system.  W = exp(lw) by
    // the same function the resampling kernels use (the table exp, <= 0.52 ulp): the weights a
    // caller reads are bit-for-bit the weights smc_resample quantizes
    out[i] = what == SMC_READ_WEIGHT ? (nl.eq ? nl.weq : smc_fm::exp_nonpos_cb(l, smc_fm::kExpTab)) : l;
}

// SPEC.md:266 / SURVEY R8: threshold >= 1 always, <= 0 never, else ess/N < threshold.
__global__ void k_ess_decide(smc_wstate *st, double threshold, double *hist_row)
{
    SMC_PDL_WAIT();
    const double eon = st->ess_over_n;
    int r = threshold >= 1.0 ? 1 : (threshold <= 0.0 ? 0 : (eon < threshold ? 1 : 0));
    if (st->status) r = 0;  // never resample on a failed normalization
    st->resample = r;
    if (hist_row) { hist_row[0] = eon; hist_row[1] = (double)r; }
}

// ---------------------------------------------------------------- reduce ----
constexpr int RB = 256;
constexpr int RMAX = 8;  // columns per pass

__global__ void __launch_bounds__(RB) k_wsum_pass(const double *__restrict__ vals, int64_t ld, int m0, int mc,
                                                   const double *__restrict__ lw_raw, const smc_wstate *st,
                                                   int64_t n, double *__restrict__ parts, int mtot)
{
    SMC_PDL_WAIT();
    __shared__ double sm[RB / 32][RMAX];
    double acc[RMAX];
#pragma unroll
    for (int j = 0; j < RMAX; ++j) acc[j] = 0.0;
    const NormLw nl = norm_of(st);
    const double w_eq = nl.weq;  // 1 / N_total after set_equal_weight
    for (int64_t i = (int64_t)blockIdx.x * RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        const double w = nl.eq ? w_eq : exp(nl(lw_raw[i]));
#pragma unroll
        for (int j = 0; j < RMAX; ++j)
            if (j < mc) acc[j] += w * vals[i * ld + m0 + j];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
        double v = warp_sum(acc[j]);
        if (lane == 0) sm[warp][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < mc) {
        double v = 0.0;
        for (int w = 0; w < RB / 32; ++w) v += sm[w][threadIdx.x];
        parts[(int64_t)blockIdx.x * mtot + m0 + threadIdx.x] = v;
    }
}

__global__ void k_wsum_final(const double *__restrict__ parts, int nb, int m, double *__restrict__ out)
{
    SMC_PDL_WAIT();
    // one warp per column, fixed order
    const int j = blockIdx.x;
    double v = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) v += parts[(int64_t)b * m + j];
    v = warp_sum(v);
    if (threadIdx.x == 0) out[j] = v;
}

inline int reduce_blocks(int64_t n)
{
    int64_t g = (n + RB - 1) / RB;
    return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

}  // namespace

size_t smc_lse_scratch_bytes() { return FG * (sizeof(LsePartial) + sizeof(double2)); }

void smc_launch_lse_finalize(const LsePartial *parts, int nparts, smc_wstate *st, int64_t n, int mode,
                             int accumulate_nc, cudaStream_t s, void *scratch, const double2 *mon_parts,
                             double *mon_out, double *partial_out)
{
    LsePartial *l2 = (LsePartial *)scratch;
    double2 *l2mon = (double2 *)(l2 + FG);
    smc_launch(k_lse_reduce, FG, FB, 0, s, parts, nparts, mon_parts, l2, l2mon, st, n, mode, accumulate_nc, mon_out,
               partial_out);
}

// One step of a captured sampler loop's bookkeeping (core.Sampler._iterate_graph), one launch
// instead of four framework kernels per step: the previous step's history row (its fused
// monitor now complete) into the history at the device cursor t - 1, the cursor advanced, and
// the next step's observation gathered into the fixed buffer the captured move reads.
__global__ void k_graph_advance(const double *__restrict__ obs, int64_t nobs, double *__restrict__ obs_out,
                                const double *__restrict__ row_prev, double *__restrict__ hist, int64_t ncols,
                                int64_t *t)
{
    SMC_PDL_WAIT();
    const int64_t tc = *t;
    __syncthreads();
    for (int64_t c = threadIdx.x; c < ncols; c += blockDim.x) hist[(tc - 1) * ncols + c] = row_prev[c];
    if (threadIdx.x < 2 && tc + 1 < nobs) obs_out[threadIdx.x] = obs[2 * (tc + 1) + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) *t = tc + 1;
}

extern "C" int smc_graph_advance(const double *obs, int64_t nobs, double *obs_out, const double *row_prev,
                                 double *hist, int64_t ncols, int64_t *t, void *stream)
{
    if (!obs || nobs < 1 || !obs_out || !row_prev || !hist || ncols < 1 || ncols > 1024 || !t)
        return smc_set_error(SMC_EINVAL, "smc_graph_advance: bad args");
    smc_launch(k_graph_advance, 1, 64, 0, (cudaStream_t)stream, obs, nobs, obs_out, row_prev, hist, ncols, t);
    return smc_check_launch("smc_graph_advance");
}

extern "C" int smc_weights_combine(const double *partials, int G, smc_wstate *st, int64_t n_total, int mode,
                                   int accumulate_nc, double *monitor_out, void *stream)
{
    if (!partials || G < 1 || !st || n_total < 1)
        return smc_set_error(SMC_EINVAL, "smc_weights_combine: bad args");
    smc_launch(k_lse_combine, 1, 1, 0, (cudaStream_t)stream, partials, G, st, n_total, mode, accumulate_nc, monitor_out);
    return smc_check_launch("smc_weights_combine");
}

extern "C" size_t smc_weights_workspace_bytes(int64_t n)
{
    return (size_t)((n + WB - 1) / WB + 1) * sizeof(LsePartial) + smc_lse_scratch_bytes() + 256;
}

extern "C" int smc_weights_update(int mode, double *lw_raw, const double *values, int64_t n, smc_wstate *st,
                                  int accumulate_nc, void *ws, size_t ws_bytes, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (n < 1 || n >= (int64_t)1 << 31 || !st || mode < 0 || mode > 4)
        return smc_set_error(SMC_EINVAL, "smc_weights_update: bad args (mode=%d n=%lld)", mode, (long long)n);
    if (mode == SMC_W_EQUAL) {
        smc_launch(k_set_equal, 1, 1, 0, s, st, n, nullptr);
        return smc_check_launch("smc_weights_update(equal)");
    }
    if (!lw_raw || !values) return smc_set_error(SMC_EINVAL, "smc_weights_update: null vector");
    if (ws_bytes < smc_weights_workspace_bytes(n) || !ws)
        return smc_set_error(SMC_EWORKSPACE, "smc_weights_update: workspace too small");
    const int nb = (int)((n + WB - 1) / WB);
    LsePartial *parts = (LsePartial *)ws;
    smc_launch(k_weights_pass, nb, WB, 0, s, mode, lw_raw, values, n, st, parts);
    void *scratch = (char *)ws + (((size_t)(nb + 1) * sizeof(LsePartial) + 255) & ~(size_t)255);
    smc_launch_lse_finalize(parts, nb, st, n, mode, accumulate_nc, s, scratch);
    return smc_check_launch("smc_weights_update");
}

extern "C" int smc_weights_set_equal(smc_wstate *st, int64_t n, const int32_t *gate, void *stream)
{
    if (!st || n < 1) return smc_set_error(SMC_EINVAL, "smc_weights_set_equal: bad args");
    smc_launch(k_set_equal, 1, 1, 0, (cudaStream_t)stream, st, n, gate);
    return smc_check_launch("smc_weights_set_equal");
}

extern "C" int smc_weights_read(int what, const double *lw_raw, const smc_wstate *st, int64_t n, double *out,
                                void *stream)
{
    if (n < 1 || !st || !out || !lw_raw || (what != 0 && what != 1))
        return smc_set_error(SMC_EINVAL, "smc_weights_read: bad args");
    smc_launch(k_weights_read, (unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream, what, lw_raw, st, n, out);
    return smc_check_launch("smc_weights_read");
}

extern "C" int smc_ess_decide(smc_wstate *st, int64_t n, double threshold, double *hist_row, void *stream)
{
    if (!st || n < 1) return smc_set_error(SMC_EINVAL, "smc_ess_decide: bad args");
    smc_launch(k_ess_decide, 1, 1, 0, (cudaStream_t)stream, st, threshold, hist_row);
    return smc_check_launch("smc_ess_decide");
}

extern "C" size_t smc_weighted_reduce_workspace_bytes(int64_t n, int64_t m)
{
    return (size_t)reduce_blocks(n) * (size_t)(m > 0 ? m : 1) * sizeof(double);
}

extern "C" int smc_weighted_reduce(const double *vals, int64_t ld, int64_t m, const double *lw_raw,
                                   const smc_wstate *st, int64_t n, double *out, void *ws, size_t ws_bytes,
                                   void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (n < 1 || m < 1 || ld < m || !vals || !lw_raw || !st || !out || m > 4096)
        return smc_set_error(SMC_EINVAL, "smc_weighted_reduce: bad args");  // SPEC.md:409 m=0 rejected
    if (!ws || ws_bytes < smc_weighted_reduce_workspace_bytes(n, m))
        return smc_set_error(SMC_EWORKSPACE, "smc_weighted_reduce: workspace too small");
    const int nb = reduce_blocks(n);
    double *parts = (double *)ws;
    for (int m0 = 0; m0 < m; m0 += RMAX) {
        const int mc = (int)((m - m0) < RMAX ? (m - m0) : RMAX);
        smc_launch(k_wsum_pass, nb, RB, 0, s, vals, ld, m0, mc, lw_raw, st, n, parts, (int)m);
    }
    smc_launch(k_wsum_final, (unsigned)m, 32, 0, s, parts, nb, (int)m, out);
    return smc_check_launch("smc_weighted_reduce");
}
