/*
 * smc_oracle.h -- CPU restatement of the smckit SMC hot path (TEST INFRASTRUCTURE).
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * Pinning: the RNG part follows /root/reference/pkg/src/smckit/rng.py line by
 * line and is checked bit-for-bit against golden draws produced by importing
 * that file (tests/golden/make_golden.py -> tests/golden/rng_golden.json).
 * Everything else restates SPEC.md (weights :17-112, resample :114-199,
 * core :255-377, exec :379-447, example-pf :449-517) plus the integer
 * resampling contract pinned in SURVEY.md Appendix A (SPEC leaves the CDF
 * arithmetic open).
 */
#ifndef SMC_ORACLE_H
#define SMC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.py ---- */
void orc_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]);
double orc_u01(uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1);
double orc_std_normal(uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1);
double orc_std_gamma(uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1, double shape);
void orc_fill(int kind, uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1, double shape,
              double *out, int64_t n);
/* one draw per stream for streams [first, first+n) -- the per-particle kernel pattern */
void orc_draw_streams(int kind, uint64_t *ctrs, uint64_t first, int64_t n, uint32_t k0, uint32_t k1,
                      double shape, double *out, int nthreads);

/* ---- weights ---- */
enum { ORC_W_SET_LOG = 0, ORC_W_ADD_LOG = 1, ORC_W_SET_LIN = 2, ORC_W_MUL_LIN = 3, ORC_W_EQUAL = 4 };
/* lw/w are the normalized log-weights / weights (in/out); values may be NULL for EQUAL.
 * Returns 0, or -3 on normalization failure (all -inf / NaN / all-zero). */
int orc_weights_update(int mode, double *lw, double *w, const double *values, int64_t n, double *ess);
/* log sum_i W_i exp(incw_i) */
double orc_nc_increment(const double *lw, const double *incw, int64_t n);

/* ---- resample (SPEC.md:114-199 + SURVEY Appendix A) ---- */
enum {
    ORC_MULTINOMIAL = 0, ORC_RESIDUAL = 1, ORC_STRATIFIED = 2, ORC_SYSTEMATIC = 3,
    ORC_RESIDUAL_STRATIFIED = 4, ORC_RESIDUAL_SYSTEMATIC = 5
};
/* counts (summing to m_out, normally m_out == n) from normalized W[n].
 * Uniforms come from u (n_u of them) when u != NULL,
 * else from stream `stream` of (ctrs, k0, k1), advancing ctrs[stream].
 * *draws_out = number of uniforms consumed.  Returns 0 or negative error:
 * -1 invalid argument, -2 unnormalized input, -4 not enough uniforms. */
int orc_resample_counts(int scheme, const double *w, int64_t n, int64_t m_out, uint64_t *ctrs,
                        uint64_t stream, uint32_t k0, uint32_t k1, const double *u, int64_t n_u,
                        int32_t *counts, int64_t *draws_out);
/* two-pointer sweep.  -1 if sum(counts) != n or a count < 0. */
int orc_replication_to_parents(const int32_t *counts, int64_t n, int32_t *parents);
/* rows j <- rows parents[j], simultaneous; X is n x d row-major */
void orc_copy_rows(double *x, int64_t n, int64_t d, const int32_t *parents);

/* ---- example-pf ---- */
double orc_cv_llh(double xpos, double ypos, double xobs, double yobs);
/* X is n x 4 row-major; streams 0..n-1 of ctrs; writes llh/incw[n]. */
void orc_cv_init(double *x, int64_t n, uint64_t *ctrs, uint32_t k0, uint32_t k1, const double *obs0,
                 double *llh, int nthreads);
void orc_cv_move(double *x, int64_t n, uint64_t *ctrs, uint32_t k0, uint32_t k1, const double *obs_t,
                 double *incw, int nthreads);

/* weighted monitor: est[j] = sum_i W_i * vals[i*m + j], sequential */
void orc_weighted_sum(const double *w, const double *vals, int64_t n, int64_t m, double *est);

/* Full PF sampler (SPEC.md:304-319 iterate order, F11 ESS rule at init).
 * hist rows (n_obs x 5): ess_over_n, resampled, pos.0, pos.1, log_zconst.
 * Returns 0 or a negative error. */
int orc_pf_run(int64_t n, uint64_t seed, int scheme, double threshold, const double *obs,
               int64_t n_obs, double *hist, double *x_out, double *lw_out, int nthreads);
/* One iterate() of the PF on an existing system (for bounded CPU timing). */
typedef struct orc_pf_sys {
    int64_t n;
    double *x, *lw, *w, *incw;
    uint64_t *ctrs;
    int32_t *counts, *parents;
    uint32_t k0, k1;
    int scheme;
    double threshold;
    double log_zconst;
} orc_pf_sys;
int orc_pf_step(orc_pf_sys *s, const double *obs_t, double *hist_row, int nthreads);
int orc_pf_initialize(orc_pf_sys *s, const double *obs0, double *hist_row, int nthreads);

/* ---- example-gmm ---- */
#define ORC_GMM_R 4   /* column stride: mu [0,4) lambda [4,8) omega [8,12); r <= 4 components used */
#define ORC_GMM_ROW 16
/* h6: xi kappa nu chi rho lambda_known (lambda_known > 0: every lambda_j fixed at that precision,
 * no Gamma prior term and no lambda move -- the conjugate-oracle model) */
double orc_gmm_llh(const double *row, int r, const double *y, int nd);
double orc_gmm_lprior(const double *row, int r, const double *h6);
void orc_gmm_init(double *x, int64_t n, int r, uint64_t *ctrs, uint32_t k0, uint32_t k1, const double *y, int nd,
                  const double *h6, int nthreads);
int64_t orc_gmm_mh(int block, double *x, int64_t n, int r, uint64_t *ctrs, uint32_t k0, uint32_t k1,
                   const double *y, int nd, const double *h6, double alpha, double sd, int nthreads);
int orc_gmm_run(int64_t n, int r, uint64_t seed, int scheme, double threshold, const double *y, int nd,
                const double *h6, int T, double power, double *hist, int nthreads);
int orc_gmm_run_steps(int64_t n, int r, uint64_t seed, int scheme, double threshold, const double *y, int nd,
                      const double *h6, int T, int steps, double power, double *hist, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
