/*
 * smc_oracle.c -- CPU restatement of the smckit SMC hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the product).  Loaded by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 *
 * Build: oracle/Makefile  (gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp).
 * -ffp-contract=off reproduces the reference's numba code, which has no FMA
 * contraction; log/cos/pow/sqrt come from glibc libm exactly
 * as numba's llvm.log.f64 / llvm.cos.f64 / llvm.pow.f64 lower to on Linux.
 */
#include "smc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------- */
/* rng.py                                                                    */
/* ------------------------------------------------------------------------- */

/* rng.py:48-54 round multipliers and Weyl key increments */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u
#define INV53 (1.0 / 9007199254740992.0) /* rng.py:55 */
#define TWO_PI (2.0 * 3.141592653589793) /* rng.py:56  2.0 * math.pi */

/* rng.py:59-72 -- _philox_block: ten rounds, key bumped after each round */
void orc_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += PHILOX_W0;
        k1 += PHILOX_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.py:75-82 -- counter (c_lo, c_hi, i_lo, i_hi); 53 bits from words 0,1 */
double orc_u01(uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1)
{
    uint64_t c = ctrs[i];
    ctrs[i] = c + 1;
    uint32_t ctr[4] = {(uint32_t)c, (uint32_t)(c >> 32), (uint32_t)i, (uint32_t)(i >> 32)};
    uint32_t w[4];
    orc_philox4x32_10(ctr, k0, k1, w);
    return ((double)(w[0] >> 5) * 67108864.0 + (double)(w[1] >> 6)) * INV53;
}

/* rng.py:85-91 -- Box-Muller cosine branch on 1 - u1 */
double orc_std_normal(uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1)
{
    double u1 = orc_u01(ctrs, i, k0, k1);
    double u2 = orc_u01(ctrs, i, k0, k1);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(TWO_PI * u2);
}

/* rng.py:94-117 -- Marsaglia-Tsang with the shape<1 boost */
double orc_std_gamma(uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1, double shape)
{
    double boost = 1.0;
    double a = shape;
    if (a < 1.0) {
        double u = 1.0 - orc_u01(ctrs, i, k0, k1);
        boost = pow(u, 1.0 / a);
        a = a + 1.0;
    }
    double d = a - 1.0 / 3.0;
    double c = 1.0 / sqrt(9.0 * d);
    for (;;) {
        double x = orc_std_normal(ctrs, i, k0, k1);
        double t = 1.0 + c * x;
        if (t <= 0.0) continue;
        double v = t * t * t;
        double u = 1.0 - orc_u01(ctrs, i, k0, k1);
        if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return boost * d * v;
    }
}

static double draw(int kind, uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1, double shape)
{
    switch (kind) {
    case 0: return orc_u01(ctrs, i, k0, k1);
    case 1: return orc_std_normal(ctrs, i, k0, k1);
    default: return orc_std_gamma(ctrs, i, k0, k1, shape);
    }
}

/* rng.py:120-135 -- fill_* : n consecutive draws from one stream */
void orc_fill(int kind, uint64_t *ctrs, uint64_t i, uint32_t k0, uint32_t k1, double shape,
              double *out, int64_t n)
{
    for (int64_t j = 0; j < n; ++j) out[j] = draw(kind, ctrs, i, k0, k1, shape);
}

void orc_draw_streams(int kind, uint64_t *ctrs, uint64_t first, int64_t n, uint32_t k0, uint32_t k1,
                      double shape, double *out, int nthreads)
{
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t j = 0; j < n; ++j) out[j] = draw(kind, ctrs, first + (uint64_t)j, k0, k1, shape);
    (void)nthreads;
}

/* ------------------------------------------------------------------------- */
/* weights                                                  */
/* ------------------------------------------------------------------------- */

/* Normalize raw log values v into lw/w (SPEC.md:96 max-shift + log-sum-exp,
 * SPEC.md:99 index-ascending sequential sums). */
static int normalize_log(const double *v, double *lw, double *w, int64_t n, double *ess)
{
    double m = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        if (isnan(v[i])) return -3;
        if (v[i] == INFINITY) return -3;
        if (v[i] > m) m = v[i];
    }
    if (m == -INFINITY) return -3; /* SPEC.md:45 all -inf */
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += exp(v[i] - m);
    double ls = log(s);
    double s2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double l = (v[i] - m) - ls;
        lw[i] = l;
        w[i] = exp(l);
        s2 += w[i] * w[i];
    }
    *ess = 1.0 / s2;
    return 0;
}

static int normalize_lin(const double *v, double *lw, double *w, int64_t n, double *ess)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (!(v[i] >= 0.0) || v[i] == INFINITY) return -3;
        s += v[i];
    }
    if (!(s > 0.0)) return -3; /* SPEC.md:65 all-zero */
    double s2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        w[i] = v[i] / s;
        lw[i] = log(w[i]);
        s2 += w[i] * w[i];
    }
    *ess = 1.0 / s2;
    return 0;
}

int orc_weights_update(int mode, double *lw, double *w, const double *values, int64_t n, double *ess)
{
    if (n < 1) return -1;
    int rc = 0;
    double *tmp = NULL;
    switch (mode) {
    case ORC_W_EQUAL:
        for (int64_t i = 0; i < n; ++i) { w[i] = 1.0 / (double)n; lw[i] = -log((double)n); }
        *ess = (double)n;
        return 0;
    case ORC_W_SET_LOG:
        return normalize_log(values, lw, w, n, ess);
    case ORC_W_ADD_LOG:
        tmp = (double *)malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) tmp[i] = lw[i] + values[i];
        rc = normalize_log(tmp, lw, w, n, ess);
        free(tmp);
        return rc;
    case ORC_W_SET_LIN:
        return normalize_lin(values, lw, w, n, ess);
    case ORC_W_MUL_LIN:
        tmp = (double *)malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) tmp[i] = w[i] * values[i];
        rc = normalize_lin(tmp, lw, w, n, ess);
        free(tmp);
        return rc;
    default:
        return -1;
    }
}

/* SPEC.md:334-341 : log sum_i W_{t-1,i} exp(incw_i), via log-sum-exp */
double orc_nc_increment(const double *lw, const double *incw, int64_t n)
{
    double m = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        double a = lw[i] + incw[i];
        if (a > m) m = a;
    }
    if (m == -INFINITY) return -INFINITY;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += exp((lw[i] + incw[i]) - m);
    return m + log(s);
}

/* ------------------------------------------------------------------------- */
/* resample under the pinned integer contract              */
/*           */
/* ------------------------------------------------------------------------- */

#define TWO63 9223372036854775808.0
#define T_LO ((((uint64_t)1) << 63) - (((uint64_t)1) << 43))
#define T_HI ((((uint64_t)1) << 63) + (((uint64_t)1) << 43))

/* A.1 quantization q_i = floor(W_i 2^63); validity window |T - 2^63| <= 2^43 */
static int quantize(const double *w, int64_t n, uint64_t *q, uint64_t *T)
{
    u128 s = 0;
    for (int64_t i = 0; i < n; ++i) {
        double wi = w[i];
        if (!(wi >= 0.0 && wi <= 1.0)) return -2;
        uint64_t qi = (uint64_t)(wi * TWO63);
        q[i] = qi;
        s += qi;
    }
    if (s < (u128)T_LO || s > (u128)T_HI) return -2;
    *T = (uint64_t)s;
    return 0;
}

static int m53(const double *u, int64_t k, uint64_t *ctrs, uint64_t stream, uint32_t k0, uint32_t k1,
               uint64_t *m)
{
    double uk = u ? u[k] : orc_u01(ctrs, stream, k0, k1);
    if (!(uk >= 0.0 && uk < 1.0)) return -1;
    *m = (uint64_t)(uk * 9007199254740992.0); /* exact: u is a multiple of 2^-53 from rng.py:82 */
    return 0;
}

/* A.2: P_k = floor((k + m_k/2^53) T / M) = a + floor((b 2^53 + m_k T) / (M 2^53)), kT = aM + b */
static uint64_t strat_pos(uint64_t k, uint64_t m, uint64_t T, uint64_t M)
{
    u128 kT = (u128)k * T;
    u128 a = kT / M, b = kT % M;
    u128 num = (b << 53) + (u128)m * T;
    return (uint64_t)(a + num / ((u128)M << 53));
}

static int cmp_u64(const void *x, const void *y)
{
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* Add, for every position p in pos[0..M) (non-decreasing), one count to the i
 * with Q_{i-1} <= p < Q_i, where Q is the inclusive prefix of q (strict upper
 * bound). */
static void sweep_add(const uint64_t *q, int64_t n, const uint64_t *pos, int64_t M, int32_t *counts)
{
    uint64_t Q = 0;
    int64_t k = 0;
    for (int64_t i = 0; i < n && k < M; ++i) {
        Q += q[i];
        while (k < M && pos[k] < Q) { counts[i] += 1; ++k; }
    }
    /* positions are < T by construction, so every k is assigned */
}

int orc_resample_counts(int scheme, const double *w, int64_t n, int64_t m_out, uint64_t *ctrs,
                        uint64_t stream, uint32_t k0, uint32_t k1, const double *u, int64_t n_u,
                        int32_t *counts, int64_t *draws_out)
{
    if (n < 1 || n > 0x7fffffffLL || scheme < 0 || scheme > 5) return -1;
    if (m_out < 1 || m_out > 0x7fffffffLL) return -1;
    *draws_out = 0;
    uint64_t *q = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    uint64_t T;
    int rc = quantize(w, n, q, &T);
    if (rc) { free(q); return rc; }
    memset(counts, 0, sizeof(int32_t) * (size_t)n);
    if (n == 1) { counts[0] = (int32_t)m_out; free(q); return 0; } /* SPEC.md:363 no-op, no draws */

    int64_t M = m_out;
    uint64_t Tm = T;
    const uint64_t *qm = q;
    uint64_t *qr = NULL;
    int residual = (scheme == ORC_RESIDUAL || scheme == ORC_RESIDUAL_STRATIFIED ||
                    scheme == ORC_RESIDUAL_SYSTEMATIC);
    if (residual) {
        /* A.4: f_i = floor(fl(N W_i)), r_i = fl(N W_i) - f_i, q'_i = floor(r_i 2^(63-L)) */
        int L = 0;
        while (((int64_t)1 << L) < n) ++L;
        double scale = ldexp(1.0, 63 - L);
        qr = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
        int64_t fsum = 0;
        uint64_t tr = 0;
        for (int64_t i = 0; i < n; ++i) {
            double x = (double)m_out * w[i];
            double f = floor(x);
            counts[i] = (int32_t)f;
            fsum += (int64_t)f;
            qr[i] = (uint64_t)((x - f) * scale);
            tr += qr[i];
        }
        M = m_out - fsum;
        if (M < 0) { free(q); free(qr); return -2; }
        if (M == 0) { free(q); free(qr); return 0; } /* (5,3,2) golden: no draws */
        if (tr == 0) { free(q); free(qr); return -2; }
        Tm = tr;
        qm = qr;
    }

    int64_t need;
    if (scheme == ORC_SYSTEMATIC || scheme == ORC_RESIDUAL_SYSTEMATIC) need = 1;
    else need = M;
    if (u && n_u < need) { free(q); free(qr); return -4; }

    uint64_t *pos = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)M);
    rc = 0;
    if (scheme == ORC_MULTINOMIAL || scheme == ORC_RESIDUAL) {
        /* A.3: P_k = floor(m_k T / 2^53), counts are order-independent */
        for (int64_t k = 0; k < M && !rc; ++k) {
            uint64_t m = 0;
            rc = m53(u, k, ctrs, stream, k0, k1, &m);
            pos[k] = (uint64_t)(((u128)m * Tm) >> 53);
        }
        if (!rc) qsort(pos, (size_t)M, sizeof(uint64_t), cmp_u64);
    } else if (scheme == ORC_STRATIFIED || scheme == ORC_RESIDUAL_STRATIFIED) {
        for (int64_t k = 0; k < M && !rc; ++k) {
            uint64_t m = 0;
            rc = m53(u, k, ctrs, stream, k0, k1, &m);
            pos[k] = strat_pos((uint64_t)k, m, Tm, (uint64_t)M);
        }
    } else { /* systematic: one uniform shared by all strata */
        uint64_t m = 0;
        rc = m53(u, 0, ctrs, stream, k0, k1, &m);
        for (int64_t k = 0; k < M && !rc; ++k) pos[k] = strat_pos((uint64_t)k, m, Tm, (uint64_t)M);
    }
    if (!rc) {
        sweep_add(qm, n, pos, M, counts);
        *draws_out = need;
    }
    free(pos);
    free(q);
    free(qr);
    return rc;
}

/* survivors keep their slot; zero-count slots, ascending,
 * take the surplus children of parents in ascending order (two pointers). */
int orc_replication_to_parents(const int32_t *counts, int64_t n, int32_t *parents)
{
    int64_t tot = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (counts[i] < 0) return -1;
        tot += counts[i];
    }
    if (tot != n) return -1;
    int64_t p = 0;      /* parent pointer */
    int64_t used = 0;   /* surplus children of p already placed */
    for (int64_t j = 0; j < n; ++j) {
        if (counts[j] >= 1) { parents[j] = (int32_t)j; continue; }
        while (counts[p] - 1 - used <= 0) { ++p; used = 0; }
        parents[j] = (int32_t)p;
        ++used;
    }
    return 0;
}

void orc_copy_rows(double *x, int64_t n, int64_t d, const int32_t *parents)
{
    double *snap = (double *)malloc(sizeof(double) * (size_t)(n * d));
    memcpy(snap, x, sizeof(double) * (size_t)(n * d));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t c = 0; c < d; ++c) x[j * d + c] = snap[(int64_t)parents[j] * d + c];
    free(snap);
}

/* ------------------------------------------------------------------------- */
/* example-pf                                                                */
/* ------------------------------------------------------------------------- */

/* PAPER.md:1181-1191 / SPEC.md:464-472 */
double orc_cv_llh(double xpos, double ypos, double xobs, double yobs)
{
    const double scale = 10;
    const double nu = 10;
    double llh_x = scale * (xpos - xobs);
    double llh_y = scale * (ypos - yobs);
    llh_x = log(1 + llh_x * llh_x / nu);
    llh_y = log(1 + llh_y * llh_y / nu);
    return -0.5 * (nu + 1) * (llh_x + llh_y);
}

/* PAPER.md:1234-1255 / SPEC.md:473-480; normal(mean, sd) = mean + sd*z (rng.py:201) */
void orc_cv_init(double *x, int64_t n, uint64_t *ctrs, uint32_t k0, uint32_t k1, const double *obs0,
                 double *llh, int nthreads)
{
    const double sd_pos0 = 2;
    const double sd_vel0 = 1;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double *r = x + 4 * i;
        r[0] = 0.0 + sd_pos0 * orc_std_normal(ctrs, (uint64_t)i, k0, k1);
        r[1] = 0.0 + sd_pos0 * orc_std_normal(ctrs, (uint64_t)i, k0, k1);
        r[2] = 0.0 + sd_vel0 * orc_std_normal(ctrs, (uint64_t)i, k0, k1);
        r[3] = 0.0 + sd_vel0 * orc_std_normal(ctrs, (uint64_t)i, k0, k1);
        llh[i] = orc_cv_llh(r[0], r[1], obs0[0], obs0[1]);
    }
    (void)nthreads;
}

/* PAPER.md:1297-1328 / SPEC.md:481-488 */
void orc_cv_move(double *x, int64_t n, uint64_t *ctrs, uint32_t k0, uint32_t k1, const double *obs_t,
                 double *incw, int nthreads)
{
    const double sd_pos = sqrt(0.02);
    const double sd_vel = sqrt(0.001);
    const double delta = 0.1;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double *r = x + 4 * i;
        r[0] = r[0] + ((0.0 + sd_pos * orc_std_normal(ctrs, (uint64_t)i, k0, k1)) + delta * r[2]);
        r[1] = r[1] + ((0.0 + sd_pos * orc_std_normal(ctrs, (uint64_t)i, k0, k1)) + delta * r[3]);
        r[2] = r[2] + (0.0 + sd_vel * orc_std_normal(ctrs, (uint64_t)i, k0, k1));
        r[3] = r[3] + (0.0 + sd_vel * orc_std_normal(ctrs, (uint64_t)i, k0, k1));
        incw[i] = orc_cv_llh(r[0], r[1], obs_t[0], obs_t[1]);
    }
    (void)nthreads;
}

void orc_weighted_sum(const double *w, const double *vals, int64_t n, int64_t m, double *est)
{
    for (int64_t j = 0; j < m; ++j) est[j] = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) est[j] += w[i] * vals[i * m + j];
}

/* ------------------------------------------------------------------------- */
/* Sampler loop for the PF                   */
/* ------------------------------------------------------------------------- */

static int resample_rule(double ess_over_n, double threshold)
{
    if (threshold >= 1.0) return 1; /* SPEC.md:266 every iteration */
    if (threshold <= 0.0) return 0; /* SPEC.md:266 never */
    return ess_over_n < threshold;
}

static int after_weights(orc_pf_sys *s, double ess, double *hist_row)
{
    int64_t n = s->n;
    double eon = ess / (double)n;
    int rs = resample_rule(eon, s->threshold);
    hist_row[0] = eon;
    hist_row[1] = rs;
    if (rs && n > 1) {
        int64_t draws;
        int rc = orc_resample_counts(s->scheme, s->w, n, n, s->ctrs, (uint64_t)n, s->k0, s->k1, NULL,
                                     0, s->counts, &draws);
        if (rc) return rc;
        rc = orc_replication_to_parents(s->counts, n, s->parents);
        if (rc) return rc;
        orc_copy_rows(s->x, n, 4, s->parents);
        orc_weights_update(ORC_W_EQUAL, s->lw, s->w, NULL, n, &ess);
    }
    /* monitor "pos", evaluated after resampling */
    double e0 = 0.0, e1 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        e0 += s->w[i] * s->x[4 * i];
        e1 += s->w[i] * s->x[4 * i + 1];
    }
    hist_row[2] = e0;
    hist_row[3] = e1;
    return 0;
}

int orc_pf_initialize(orc_pf_sys *s, const double *obs0, double *hist_row, int nthreads)
{
    double ess;
    orc_cv_init(s->x, s->n, s->ctrs, s->k0, s->k1, obs0, s->incw, nthreads);
    /* log Z_0 = log (1/N) sum_i exp(llh_i): the equal-weight prior sample weighted once */
    for (int64_t i = 0; i < s->n; ++i) s->lw[i] = -log((double)s->n);
    s->log_zconst = orc_nc_increment(s->lw, s->incw, s->n);
    int rc = orc_weights_update(ORC_W_SET_LOG, s->lw, s->w, s->incw, s->n, &ess);
    if (rc) return rc;
    hist_row[4] = s->log_zconst;
    return after_weights(s, ess, hist_row); /* F11: ESS rule applied after init */
}

int orc_pf_step(orc_pf_sys *s, const double *obs_t, double *hist_row, int nthreads)
{
    double ess;
    orc_cv_move(s->x, s->n, s->ctrs, s->k0, s->k1, obs_t, s->incw, nthreads);
    s->log_zconst += orc_nc_increment(s->lw, s->incw, s->n);
    int rc = orc_weights_update(ORC_W_ADD_LOG, s->lw, s->w, s->incw, s->n, &ess);
    if (rc) return rc;
    hist_row[4] = s->log_zconst;
    return after_weights(s, ess, hist_row);
}

int orc_pf_run(int64_t n, uint64_t seed, int scheme, double threshold, const double *obs,
               int64_t n_obs, double *hist, double *x_out, double *lw_out, int nthreads)
{
    orc_pf_sys s;
    s.n = n;
    s.x = (double *)malloc(sizeof(double) * (size_t)(4 * n));
    s.lw = (double *)malloc(sizeof(double) * (size_t)n);
    s.w = (double *)malloc(sizeof(double) * (size_t)n);
    s.incw = (double *)malloc(sizeof(double) * (size_t)n);
    s.ctrs = (uint64_t *)calloc((size_t)(n + 1), sizeof(uint64_t));
    s.counts = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    s.parents = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    s.k0 = (uint32_t)seed;
    s.k1 = (uint32_t)(seed >> 32);
    s.scheme = scheme;
    s.threshold = threshold;
    int rc = orc_pf_initialize(&s, obs, hist, nthreads);
    for (int64_t t = 1; t < n_obs && !rc; ++t) rc = orc_pf_step(&s, obs + 2 * t, hist + 5 * t, nthreads);
    if (!rc) {
        if (x_out) memcpy(x_out, s.x, sizeof(double) * (size_t)(4 * n));
        if (lw_out) memcpy(lw_out, s.lw, sizeof(double) * (size_t)n);
    }
    free(s.x); free(s.lw); free(s.w); free(s.incw); free(s.ctrs); free(s.counts); free(s.parents);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* example-gmm                         */
/* state row: mu[4] lambda[4] omega[4] log_prior log_likelihood pad pad       */
/* ------------------------------------------------------------------------- */

static void gmm_hyper_derive(const double *h6, int r, double *h)
{
    /* h: xi kappa nu chi rho lambda_known | lgamma(nu) log(chi) log(kappa/2pi) dirichlet_const */
    for (int k = 0; k < 6; ++k) h[k] = h6[k];
    h[6] = lgamma(h[2]);
    h[7] = log(h[3]);
    h[8] = log(h[1] / (2.0 * 3.141592653589793));
    h[9] = lgamma(r * h[4]) - r * lgamma(h[4]);
}

/* update_log_likelihood:
 * -n/2 log 2pi + sum_k log sum_{j<r} w_j exp(.5 log l_j - .5 l_j (y_k - mu_j)^2) */
double orc_gmm_llh(const double *row, int r, const double *y, int nd)
{
    double ll = -0.5 * (double)nd * 1.8378770664093455;
    double lj[ORC_GMM_R];
    for (int j = 0; j < r; ++j) lj[j] = log(row[ORC_GMM_R + j]);
    for (int k = 0; k < nd; ++k) {
        double lli = 0;
        for (int j = 0; j < r; ++j) {
            double resid = y[k] - row[j];
            lli += row[2 * ORC_GMM_R + j] * exp(0.5 * lj[j] - 0.5 * row[ORC_GMM_R + j] * resid * resid);
        }
        ll += log(lli);
    }
    return ll;
}

/* update_log_prior: Normal(xi, 1/kappa) per mu, Gamma(nu, scale chi) per lambda
 * (absent when lambda is known), symmetric Dirichlet(rho) on omega */
double orc_gmm_lprior(const double *row, int r, const double *h6)
{
    double h[10];
    gmm_hyper_derive(h6, r, h);
    double lp = 0;
    for (int j = 0; j < r; ++j) {
        double d = row[j] - h[0];
        lp += h[8] * 0.5 - 0.5 * h[1] * d * d;
        if (!(h[5] > 0)) {
            double lam = row[ORC_GMM_R + j];
            lp += (h[2] - 1) * log(lam) - lam / h[3] - h[6] - h[2] * h[7];
        }
        if (h[4] != 1.0) lp += (h[4] - 1) * log(row[2 * ORC_GMM_R + j]);
    }
    return lp + h[9];
}

/* gmm_init::initialize_state for particles [0, n): per component in
 * order mu ~ N(xi, 1/kappa), lambda ~ Gamma(nu, chi) (unless known), omega ~ Gamma(1, 1);
 * normalize omega */
void orc_gmm_init(double *x, int64_t n, int r, uint64_t *ctrs, uint32_t k0, uint32_t k1, const double *y, int nd,
                  const double *h6, int nthreads)
{
    const double sd0 = 1.0 / sqrt(h6[1]);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double *row = x + ORC_GMM_ROW * i;
        double sum = 0;
        memset(row, 0, sizeof(double) * ORC_GMM_ROW);
        for (int j = 0; j < r; ++j) {
            row[j] = h6[0] + sd0 * orc_std_normal(ctrs, (uint64_t)i, k0, k1);
            row[ORC_GMM_R + j] = h6[5] > 0 ? h6[5] : h6[3] * orc_std_gamma(ctrs, (uint64_t)i, k0, k1, h6[2]);
            row[2 * ORC_GMM_R + j] = 1.0 * orc_std_gamma(ctrs, (uint64_t)i, k0, k1, 1.0);
            sum += row[2 * ORC_GMM_R + j];
        }
        for (int j = 0; j < r; ++j) row[2 * ORC_GMM_R + j] /= sum;
        row[12] = orc_gmm_lprior(row, r, h6);
        row[13] = orc_gmm_llh(row, r, y, nd);
    }
    (void)nthreads;
}

/* gmm_move_{mu,lambda,weight}: returns #accepted */
int64_t orc_gmm_mh(int block, double *x, int64_t n, int r, uint64_t *ctrs, uint32_t k0, uint32_t k1,
                   const double *y, int nd, const double *h6, double alpha, double sd, int nthreads)
{
    int64_t acc = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) reduction(+ : acc) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double *row = x + ORC_GMM_ROW * i;
        double p[ORC_GMM_ROW];
        memcpy(p, row, sizeof(p));
        double p_old = row[12] + alpha * row[13];
        double jac = 0;
        if (block == 0) {
            for (int j = 0; j < r; ++j) p[j] += 0.0 + sd * orc_std_normal(ctrs, (uint64_t)i, k0, k1);
        } else if (block == 1) {
            for (int j = 0; j < r; ++j) {
                double old = p[ORC_GMM_R + j];
                p[ORC_GMM_R + j] = old * exp(0.0 + sd * orc_std_normal(ctrs, (uint64_t)i, k0, k1));
                jac += log(p[ORC_GMM_R + j]) - log(old);
            }
        } else {
            double g[ORC_GMM_R];
            double *om = p + 2 * ORC_GMM_R;
            for (int j = 0; j < r; ++j) jac -= log(om[j]);
            for (int j = 0; j < r - 1; ++j)
                g[j] = log(om[j] / om[r - 1]) + (0.0 + sd * orc_std_normal(ctrs, (uint64_t)i, k0, k1));
            g[r - 1] = 0.0;
            double gm = g[0];
            for (int j = 1; j < r; ++j) gm = fmax(gm, g[j]);
            double s = 0;
            for (int j = 0; j < r; ++j) { om[j] = exp(g[j] - gm); s += om[j]; }
            for (int j = 0; j < r; ++j) { om[j] /= s; jac += log(om[j]); }
        }
        double lp = orc_gmm_lprior(p, r, h6), ll = orc_gmm_llh(p, r, y, nd);
        double dp = lp + alpha * ll - p_old + jac;
        double u = log(orc_u01(ctrs, (uint64_t)i, k0, k1));
        if (u < dp) {
            p[12] = lp;
            p[13] = ll;
            memcpy(row, p, sizeof(p));
            acc += 1;
        }
    }
    (void)nthreads;
    return acc;
}

/* The GMM sampler: prior annealing
 * alpha_t = (t/T)^power, move_smc -> ESS rule -> resample -> mu, lambda (unless known),
 * weight (r > 1) MH -> path (alpha_t, sum W llh).  hist rows (T+1) x 8: ess_over_n resampled
 * acc_mu acc_lambda acc_weight alpha U_t log_zconst. */
int orc_gmm_run(int64_t n, int r, uint64_t seed, int scheme, double threshold, const double *y, int nd,
                const double *h6, int T, double power, double *hist, int nthreads)
{
    return orc_gmm_run_steps(n, r, seed, scheme, threshold, y, nd, h6, T, T, power, hist, nthreads);
}

/* The first `steps` iterations of a T-iteration run (the alpha schedule is T's). */
int orc_gmm_run_steps(int64_t n, int r, uint64_t seed, int scheme, double threshold, const double *y, int nd,
                      const double *h6, int T, int steps, double power, double *hist, int nthreads)
{
    double *x = (double *)calloc((size_t)(ORC_GMM_ROW * n), sizeof(double));
    double *lw = (double *)malloc(sizeof(double) * (size_t)n), *w = (double *)malloc(sizeof(double) * (size_t)n);
    double *incw = (double *)malloc(sizeof(double) * (size_t)n);
    uint64_t *ctrs = (uint64_t *)calloc((size_t)(n + 1), sizeof(uint64_t));
    int32_t *counts = (int32_t *)malloc(sizeof(int32_t) * (size_t)n), *parents = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    double ess, alpha = 0.0, log_z = 0.0;
    int rc = 0;
    const int use[3] = {1, !(h6[5] > 0), r > 1};
    orc_gmm_init(x, n, r, ctrs, k0, k1, y, nd, h6, nthreads);
    orc_weights_update(ORC_W_EQUAL, lw, w, NULL, n, &ess);
    for (int t = 0; t <= steps && t <= T && !rc; ++t) {
        double *hr = hist + 8 * t;
        double acc[3] = {0, 0, 0};
        if (t > 0) {
            double a = pow((double)t / (double)T, power);
            a = a < 1 ? a : 1;
            a = a > 0 ? a : 0;
            double dalpha = a - alpha;
            alpha = a;
            double ac = alpha < 0.02 ? 0.02 : alpha;
            double sds[3] = {0.15 / ac, (1 + sqrt(1 / ac)) * 0.15, (1 + sqrt(1 / ac)) * 0.2};
            for (int64_t i = 0; i < n; ++i) incw[i] = dalpha * x[ORC_GMM_ROW * i + 13];
            log_z += orc_nc_increment(lw, incw, n);
            rc = orc_weights_update(ORC_W_ADD_LOG, lw, w, incw, n, &ess);
            if (rc) break;
            double eon = ess / (double)n;
            int rs = resample_rule(eon, threshold);
            hr[0] = eon;
            hr[1] = rs;
            if (rs && n > 1) {
                int64_t draws;
                rc = orc_resample_counts(scheme, w, n, n, ctrs, (uint64_t)n, k0, k1, NULL, 0, counts, &draws);
                if (!rc) rc = orc_replication_to_parents(counts, n, parents);
                if (rc) break;
                orc_copy_rows(x, n, ORC_GMM_ROW, parents);
                orc_weights_update(ORC_W_EQUAL, lw, w, NULL, n, &ess);
            }
            for (int b = 0; b < 3; ++b)
                if (use[b]) acc[b] = (double)orc_gmm_mh(b, x, n, r, ctrs, k0, k1, y, nd, h6, alpha, sds[b], nthreads);
        } else {
            hr[0] = ess / (double)n;
            hr[1] = resample_rule(hr[0], threshold);
        }
        double u = 0;
        for (int64_t i = 0; i < n; ++i) u += w[i] * x[ORC_GMM_ROW * i + 13];
        hr[2] = acc[0];
        hr[3] = acc[1];
        hr[4] = acc[2];
        hr[5] = alpha;
        hr[6] = u;
        hr[7] = log_z;
    }
    free(x); free(lw); free(w); free(incw); free(ctrs); free(counts); free(parents);
    return rc;
}
