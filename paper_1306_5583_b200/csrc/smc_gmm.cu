// smc_gmm.cu -- the paper's Gaussian-mixture SMC sampler (
// PAPER.md:1516-1981; config 3): tempered targets pi_alpha ∝ prior * lik^alpha,
// three-block random-walk Metropolis moves, direct (NC) and path-sampling log Z.
//
// State: N x 16 f64 row-major (128 B = 4 sectors per particle):
//   [0,4) mu, [4,8) lambda, [8,12) omega, 12 log_prior, 13 log_likelihood.
// The data (n <= 4096 doubles) is staged once per block in shared memory; the
// likelihood loop is the hot spot: per data point r exp + 1 log (FP64 bound).
#include "smc_weights.cuh"

using namespace smc;

namespace {

constexpr int GB = 128;  // threads per block (register-heavy per-particle loops)
#ifndef GMM_MIN_BLOCKS
#define GMM_MIN_BLOCKS 4
#endif
constexpr int RS = 4;    // column stride of mu / lambda / omega in a row (SMC_GMM_MAX_R)
constexpr int W = SMC_GMM_ROW;

struct Hyper {
    double xi, kappa, nu, chi, rho, lambda_known;
    double lgamma_nu, log_chi, log_kappa_2pi, dir_const;
};

template <int R>
struct Param {
    double mu[R], lam[R], om[R];
};

template <int R>
SMC_DEV void load_param(const double *row, Param<R> &p)
{
#pragma unroll
    for (int j = 0; j < R; ++j) { p.mu[j] = row[j]; p.lam[j] = row[RS + j]; p.om[j] = row[2 * RS + j]; }
}

template <int R>
SMC_DEV void store_param(double *row, const Param<R> &p)
{
#pragma unroll
    for (int j = 0; j < R; ++j) { row[j] = p.mu[j]; row[RS + j] = p.lam[j]; row[2 * RS + j] = p.om[j]; }
}

// update_log_likelihood: -n/2 log 2pi + sum_k log sum_j w_j exp(.5 log l_j - .5 l_j r^2).
// Evaluated per point k as  x_j = c_j + b_j r_j^2  (c_j = .5 log l_j + log w_j, b_j = -l_j / 2),
// m = max_j x_j,  log sum_j exp(x_j) = m + log S,  S = sum_j exp(x_j - m) in [1, R]:
// the max-shifted terms never overflow, anything below 2^-1022 is far under S's rounding
// (exp_nonpos flushes it), and a point far from every component keeps its exact, finite
// log density.  sum_k m_k is a plain running sum; prod_k S_k one log of a renormalized
// running product (S_k >= 1: no checks).  Per (point, component) ~13 fp64 ops.  Agrees
// with the oracle's sum of libm logs to ~1e-12 relative.  Non-finite parameters take the
// direct evaluation (log_likelihood_direct) so NaN / inf propagate as in the reference.
template <int R>
SMC_DEV double log_likelihood_direct(const Param<R> &p, const double *__restrict__ y, int nd)
{
    double ll = -0.5 * (double)nd * 1.8378770664093455;
    for (int k = 0; k < nd; ++k) {
        double lli = 0;
        for (int j = 0; j < R; ++j) {
            const double resid = y[k] - p.mu[j];
            lli += p.om[j] * exp(0.5 * log(p.lam[j]) - 0.5 * p.lam[j] * resid * resid);
        }
        ll += log(lli);
    }
    return ll;
}

// The exp table in shared memory as TAB_COPIES interleaved copies (entry k of copy c at
// k * TAB_COPIES + c; each thread reads copy threadIdx % TAB_COPIES): an LDS.128 serves a
// warp in phases of 8 lanes, and 8 lanes reading 8 different copies hit 8 different bank
// groups -- the random exp indices no longer conflict (the single table measured 764 M of
// 1322 M shared wavefronts as conflicts, profiles/r1_ncu_gmm_mh.txt).
constexpr int TAB_COPIES = 8;
constexpr int TAB_N = 256;  // exp_nonpos256's table
constexpr size_t TAB_BYTES = TAB_N * TAB_COPIES * sizeof(smc_fm::ExpEntry);

template <int R>
SMC_DEV double log_likelihood(const Param<R> &p, const double *__restrict__ y, int nd,
                              const smc_fm::ExpEntry *__restrict__ tab)
{
    double c[R], b[R];
    bool finite = true;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        c[j] = 0.5 * log(p.lam[j]) + log(p.om[j]);  // update_log_lambda
        b[j] = -0.5 * p.lam[j];
        finite = finite && isfinite(p.mu[j]) && isfinite(b[j]) && p.lam[j] > 0 && !isnan(c[j]) && c[j] < INFINITY;
    }
    if (!finite) return log_likelihood_direct(p, y, nd);
    double msum = 0.0, prod = 1.0;
    int64_t ex = 0;
    smc_fm::LogProd far;  // points whose largest term is near / below the underflow threshold
    for (int k = 0; k < nd; ++k) {
        const double yk = y[k];
        double x[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const double resid = yk - p.mu[j];
            x[j] = __fma_rn(b[j], resid * resid, c[j]);
        }
        double m = x[0];
        int im = 0;
#pragma unroll
        // plain compare-select (x is finite or -inf; fmax's NaN handling measured 5 % slower)
        for (int j = 1; j < R; ++j) {
            im = x[j] > m ? j : im;
            m = x[j] > m ? x[j] : m;
        }
        if (m >= -700.0) {
            // the largest term is exp(0) = 1 exactly: only the R - 1 others need the exp
            // (selected around the first maximum, in component order)
            double S = 1.0;
#pragma unroll
            for (int j = 0; j + 1 < R; ++j)
                S += smc_fm::exp_nonpos256((j < im ? x[j] : x[j + 1]) - m, tab, TAB_COPIES, (int)(threadIdx.x % TAB_COPIES));
            msum += m;
            prod *= S;  // prod in [1, 2) times S in [1, R]: normal; peel the exponent off
            const uint64_t pb = smc_fm::bits(prod);
            ex += (int64_t)(pb >> 52) - 1023;
            prod = smc_fm::from_bits((pb & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
        } else {
            // rare (a point far from every component): the reference's own arithmetic, terms
            // rounded into the subnormal range and a zero sum giving -inf, as libm does
            double lli = 0.0;
#pragma unroll
            for (int j = 0; j < R; ++j) lli += smc_fm::exp(x[j], smc_fm::kExpTab);
            far.add(lli);
        }
    }
    const double e = (double)ex;
    return -0.5 * (double)nd * 1.8378770664093455 + msum +
           (e * 0x1.62e42fefa3800p-1 + (smc_fm::log_core(prod) + e * 0x1.ef35793c76730p-45)) + far.result();
}

// update_log_prior: Normal(xi, 1/kappa) per mu, Gamma(nu, chi) per
// lambda (absent when lambda is known), symmetric Dirichlet(rho) for omega.
template <int R>
SMC_DEV double log_prior(const Param<R> &p, const Hyper &h)
{
    double lp = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const double d = p.mu[j] - h.xi;
        lp += h.log_kappa_2pi * 0.5 - 0.5 * h.kappa * d * d;
        if (!(h.lambda_known > 0))
            lp += (h.nu - 1) * log(p.lam[j]) - p.lam[j] / h.chi - h.lgamma_nu - h.nu * h.log_chi;
        if (h.rho != 1.0) lp += (h.rho - 1) * log(p.om[j]);
    }
    return lp + h.dir_const;
}

// Shared memory: the exp table (2 KB) then the data (nd doubles, <= 32 KB).

SMC_DEV void stage_data(const double *__restrict__ data, int nd, smc_fm::ExpEntry *s_tab, double *s_y)
{
    for (int k = threadIdx.x; k < TAB_N * TAB_COPIES; k += blockDim.x) s_tab[k] = smc_fm::kExpTab256[k / TAB_COPIES];
    for (int k = threadIdx.x; k < nd; k += blockDim.x) s_y[k] = data[k];
    __syncthreads();
}

size_t smem_bytes(int nd) { return TAB_BYTES + (size_t)nd * sizeof(double); }

// gmm_init::initialize_state: per component, in order,
// mu ~ N(mu0, sd0), lambda ~ Gamma(shape0, scale0), weight ~ Gamma(1, 1); normalize.
template <int R>
__global__ void __launch_bounds__(GB) k_gmm_init(double *__restrict__ x, int64_t n, uint64_t sbase, Key key,
                                                 uint64_t *__restrict__ ctrs, const double *__restrict__ data, int nd,
                                                 Hyper h)
{
    extern __shared__ double4 s_raw[];
    smc_fm::ExpEntry *s_tab = (smc_fm::ExpEntry *)s_raw;
    double *s_y = (double *)((char *)s_raw + TAB_BYTES);
    stage_data(data, nd, s_tab, s_y);
    const int64_t i = (int64_t)blockIdx.x * GB + threadIdx.x;
    if (i >= n) return;
    const uint64_t si = sbase + (uint64_t)i;
    uint64_t c = ctrs[i];
    Param<R> p;
    const double sd0 = 1.0 / sqrt(h.kappa);
    double sum = 0;
    for (int j = 0; j < R; ++j) {
        p.mu[j] = h.xi + sd0 * normal_at(c, si, key);
        c += 2;
        p.lam[j] = h.lambda_known > 0 ? h.lambda_known : h.chi * gamma_from(c, si, key, h.nu);
        p.om[j] = 1.0 * gamma_from(c, si, key, 1.0);
        sum += p.om[j];
    }
    for (int j = 0; j < R; ++j) p.om[j] /= sum;
    ctrs[i] = c;
    double *row = x + i * W;
    for (int j = 0; j < 12; ++j) row[j] = 0.0;
    store_param(row, p);
    row[12] = log_prior(p, h);
    row[13] = log_likelihood(p, s_y, nd, s_tab);
}

// gmm_move_smc: incw = dalpha * llh; nc_add_log_weight then
// add_log_weight -- fused with the one-pass lse partials.
__global__ void __launch_bounds__(256) k_gmm_reweight(const double *__restrict__ x, double *__restrict__ lw_raw,
                                                      int64_t n, double dalpha, smc_wstate *st,
                                                      LsePartial *__restrict__ parts)
{
    const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    double v = -INFINITY;
    if (i < n) {
        const NormLw nl = norm_of(st);
        const double prev = nl(nl.needs_raw() ? lw_raw[i] : 0.0);
        v = prev + dalpha * x[i * W + 13];
        if (isnan(v) || v == INFINITY) { raise_status_at(&st->status, SMC_ENORMALIZE, i); v = -INFINITY; }
        lw_raw[i] = v;
    }
    LsePartial p = block_lse_partial<256>(v);
    if (threadIdx.x == 0) parts[blockIdx.x] = p;
}

// gmm_move_mu / _lambda / _weight: random walk,
// recompute caches, accept iff log U < p_new - p_old (+ Jacobian).  Draws: the block's
// normals in component order, then one uniform.
template <int BLOCK, int R>
__global__ void __launch_bounds__(GB, GMM_MIN_BLOCKS) k_gmm_mh(double *__restrict__ x, int64_t n, uint64_t sbase, Key key,
                                               uint64_t *__restrict__ ctrs, const double *__restrict__ data, int nd,
                                               Hyper h, double alpha, double sd,
                                               unsigned long long *__restrict__ accepted)
{
    extern __shared__ double4 s_raw[];
    smc_fm::ExpEntry *s_tab = (smc_fm::ExpEntry *)s_raw;
    double *s_y = (double *)((char *)s_raw + TAB_BYTES);
    stage_data(data, nd, s_tab, s_y);
    const int64_t i = (int64_t)blockIdx.x * GB + threadIdx.x;
    int acc = 0;
    if (i < n) {
        double *row = x + i * W;
        Param<R> p;
        load_param(row, p);
        const double lp_old = row[12], ll_old = row[13];
        const double p_old = lp_old + alpha * ll_old;
        const uint64_t si = sbase + (uint64_t)i;
        uint64_t c = ctrs[i];
        double jac = 0;
        if (BLOCK == 0) {  // mu_j += N(0, mu_sd)
#pragma unroll
            for (int j = 0; j < R; ++j) { p.mu[j] += 0.0 + sd * normal_at(c, si, key); c += 2; }
        } else if (BLOCK == 1) {  // log-scale walk on lambda, Jacobian sum(log l_new - log l_old)
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const double old = p.lam[j];
                p.lam[j] = old * exp(0.0 + sd * normal_at(c, si, key));
                c += 2;
                jac += log(p.lam[j]) - log(old);
            }
        } else {  // logit walk on omega (omega_R reference), Jacobian sum_j (log w_new - log w_old)
            double g[R];
#pragma unroll
            for (int j = 0; j < R; ++j) jac -= log(p.om[j]);
#pragma unroll
            for (int j = 0; j < R - 1; ++j) {
                g[j] = log(p.om[j] / p.om[R - 1]) + (0.0 + sd * normal_at(c, si, key));
                c += 2;
            }
            g[R - 1] = 0.0;
            double gm = g[0];
#pragma unroll
            for (int j = 1; j < R; ++j) gm = fmax(gm, g[j]);
            double s = 0;
#pragma unroll
            for (int j = 0; j < R; ++j) { p.om[j] = exp(g[j] - gm); s += p.om[j]; }
#pragma unroll
            for (int j = 0; j < R; ++j) { p.om[j] /= s; jac += log(p.om[j]); }
        }
        const double lp_new = log_prior(p, h);
        const double ll_new = log_likelihood(p, s_y, nd, s_tab);
        const double dp = lp_new + alpha * ll_new - p_old + jac;
        const double u = log(u01_at(c, si, key));
        c += 1;
        ctrs[i] = c;
        if (u < dp) {  // accept (strict)
            store_param(row, p);
            row[12] = lp_new;
            row[13] = ll_new;
            acc = 1;
        }
    }
    // acceptance count: block sum, one integer atomic (order-free, exact)
    __shared__ int s_acc[GB / 32];
    const int a = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) s_acc[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < GB / 32; ++w) t += s_acc[w];
        if (t) atomicAdd(accepted, (unsigned long long)t);
    }
}

// log-prior / log-likelihood of given parameter rows (the cache-coherence hook).
template <int R>
__global__ void __launch_bounds__(GB) k_gmm_eval(double *__restrict__ x, int64_t n, const double *__restrict__ data,
                                                 int nd, Hyper h)
{
    extern __shared__ double4 s_raw[];
    smc_fm::ExpEntry *s_tab = (smc_fm::ExpEntry *)s_raw;
    double *s_y = (double *)((char *)s_raw + TAB_BYTES);
    stage_data(data, nd, s_tab, s_y);
    const int64_t i = (int64_t)blockIdx.x * GB + threadIdx.x;
    if (i >= n) return;
    double *row = x + i * W;
    Param<R> p;
    load_param(row, p);
    row[12] = log_prior(p, h);
    row[13] = log_likelihood(p, s_y, nd, s_tab);
}

Hyper make_hyper(const double *hyper6, int R)
{
    Hyper h;
    h.xi = hyper6[0];
    h.kappa = hyper6[1];
    h.nu = hyper6[2];
    h.chi = hyper6[3];
    h.rho = hyper6[4];
    h.lambda_known = hyper6[5];
    h.lgamma_nu = lgamma(h.nu);
    h.log_chi = log(h.chi);
    h.log_kappa_2pi = log(h.kappa / (2.0 * 3.141592653589793));
    h.dir_const = lgamma(R * h.rho) - R * lgamma(h.rho);  // Dirichlet normalizer (ln (r-1)! at rho = 1), R = r
    return h;
}

int gmm_check(const double *x, int64_t n, int r, const double *data, int nd, const double *hyper, const char *who)
{
    if (!x || n < 1 || n >= ((int64_t)1 << 31) || !data || nd < 1 || nd > SMC_GMM_MAX_DATA || !hyper)
        return smc_set_error(SMC_EINVAL, "%s: bad args", who);
    if (r < 1 || r > SMC_GMM_MAX_R) return smc_set_error(SMC_EINVAL, "%s: r = %d outside [1, %d]", who, r, SMC_GMM_MAX_R);
    if (hyper[5] < 0 || hyper[5] != hyper[5]) return smc_set_error(SMC_EINVAL, "%s: lambda_known must be >= 0", who);
    if (!(hyper[1] > 0 && hyper[2] > 0 && hyper[3] > 0 && hyper[4] > 0))
        return smc_set_error(SMC_EINVAL, "%s: hyperparameters must be positive", who);
    return SMC_OK;
}

}  // namespace

// r -> template instantiation (r = 1..SMC_GMM_MAX_R)
// more than 48 KB of dynamic shared memory (4096 data points + the replicated exp table) needs
// the kernel's opt-in, set on every launch that asks for it (cheap, host-side)
template <class K>
inline void allow_smem(K kern, size_t bytes)
{
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

#define SMC_GMM_DISPATCH(r, CALL)          \
    switch (r) {                            \
    case 1: { constexpr int R = 1; CALL; } break; \
    case 2: { constexpr int R = 2; CALL; } break; \
    case 3: { constexpr int R = 3; CALL; } break; \
    default: { constexpr int R = 4; CALL; } break; \
    }

extern "C" int smc_gmm_init(double *x, int64_t n, int r, uint64_t stream_base, uint64_t seed, uint64_t *ctrs,
                            const double *data, int nd, const double *hyper, void *stream)
{
    int rc = gmm_check(x, n, r, data, nd, hyper, "smc_gmm_init");
    if (rc) return rc;
    if (!ctrs) return smc_set_error(SMC_EINVAL, "smc_gmm_init: ctrs");
    const Key key{(uint32_t)seed, (uint32_t)(seed >> 32)};
    const Hyper h = make_hyper(hyper, r);
    const unsigned nb = (unsigned)((n + GB - 1) / GB);
    SMC_GMM_DISPATCH(r, (allow_smem(k_gmm_init<R>, smem_bytes(nd)), k_gmm_init<R><<<nb, GB, smem_bytes(nd), (cudaStream_t)stream>>>(x, n, stream_base, key, ctrs,
                                                                                       data, nd, h)));
    SMC_COUNT_LAUNCH();
    return smc_check_launch("smc_gmm_init");
}

extern "C" int smc_gmm_eval(double *x, int64_t n, int r, const double *data, int nd, const double *hyper, void *stream)
{
    int rc = gmm_check(x, n, r, data, nd, hyper, "smc_gmm_eval");
    if (rc) return rc;
    const Hyper h = make_hyper(hyper, r);
    const unsigned nb = (unsigned)((n + GB - 1) / GB);
    SMC_GMM_DISPATCH(r, (allow_smem(k_gmm_eval<R>, smem_bytes(nd)), k_gmm_eval<R><<<nb, GB, smem_bytes(nd), (cudaStream_t)stream>>>(x, n, data, nd, h)));
    SMC_COUNT_LAUNCH();
    return smc_check_launch("smc_gmm_eval");
}

extern "C" size_t smc_gmm_workspace_bytes(int64_t n)
{
    return (size_t)((n + 255) / 256 + 1) * sizeof(LsePartial) + smc_lse_scratch_bytes() + 512;
}

extern "C" int smc_gmm_reweight(const double *x, double *lw_raw, int64_t n, double dalpha, smc_wstate *st,
                                double *partial_out, void *ws, size_t ws_bytes, void *stream)
{
    if (!x || !lw_raw || !st || n < 1 || n >= ((int64_t)1 << 31))
        return smc_set_error(SMC_EINVAL, "smc_gmm_reweight: bad args");
    if (!ws || ws_bytes < smc_gmm_workspace_bytes(n)) return smc_set_error(SMC_EWORKSPACE, "smc_gmm_reweight: ws");
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = (int)((n + 255) / 256);
    LsePartial *parts = (LsePartial *)ws;
    void *scratch = (char *)ws + (((size_t)(nb + 1) * sizeof(LsePartial) + 255) & ~(size_t)255);
    k_gmm_reweight<<<nb, 256, 0, s>>>(x, lw_raw, n, dalpha, st, parts);
    SMC_COUNT_LAUNCH();
    smc_launch_lse_finalize(parts, nb, st, n, SMC_W_ADD_LOG, 1, s, scratch, nullptr, nullptr, partial_out);
    return smc_check_launch("smc_gmm_reweight");
}

extern "C" int smc_gmm_mh(int block, double *x, int64_t n, int r, uint64_t stream_base, uint64_t seed,
                          uint64_t *ctrs, const double *data, int nd, const double *hyper, double alpha, double sd,
                          unsigned long long *accepted, void *stream)
{
    int rc = gmm_check(x, n, r, data, nd, hyper, "smc_gmm_mh");
    if (rc) return rc;
    if (!ctrs || !accepted || block < 0 || block > 2 || !(sd >= 0))
        return smc_set_error(SMC_EINVAL, "smc_gmm_mh: bad args");
    cudaStream_t s = (cudaStream_t)stream;
    const Key key{(uint32_t)seed, (uint32_t)(seed >> 32)};
    const Hyper h = make_hyper(hyper, r);
    const unsigned nb = (unsigned)((n + GB - 1) / GB);
    const size_t sm = smem_bytes(nd);
#define SMC_GMM_MH(B) \
    SMC_GMM_DISPATCH(r, (allow_smem(k_gmm_mh<B, R>, sm), k_gmm_mh<B, R><<<nb, GB, sm, s>>>(x, n, stream_base, key, ctrs, data, nd, h, alpha, sd, accepted)))
    if (block == 0) { SMC_GMM_MH(0) }
    else if (block == 1) { SMC_GMM_MH(1) }
    else { SMC_GMM_MH(2) }
#undef SMC_GMM_MH
    SMC_COUNT_LAUNCH();
    return smc_check_launch("smc_gmm_mh");
}
