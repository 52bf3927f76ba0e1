/*
 * smc_abi.h -- C ABI of the B200 (sm_100a) SMC hot path.
 *
 * Drop-in boundary for the data-parallel path of smckit / vSMC (arXiv 1306.5583).
 * The reference is a Python package whose only shipped module is
 * pkg/src/smckit/rng.py; the other modules (weights, resample, core, exec,
 * example-pf) are specified in /root/reference/SPEC.md.  Each entry point below
 * names the reference interface it replaces (file:line).  A ctypes binding of
 * this header is paper_1306_5583_b200/_abi.py; INTEGRATION.md shows the stub a
 * smckit maintainer would add.
 *
 * Conventions
 *  - Every pointer argument is DEVICE memory owned by the caller (torch CUDA
 *    tensors in the Python host), except `smc_last_error`'s buffer.  The
 *    library never allocates; scratch comes in through (ws, ws_bytes), sized by
 *    the matching *_workspace_bytes call.
 *  - Every call takes the cudaStream_t it is ordered on (passed as void*) and
 *    is asynchronous; no call synchronizes the device.
 *  - Return value: SMC_OK or a negative SMC_E* code for host-detectable
 *    failures (bad argument, launch failure).  Data-dependent failures that
 *    only the device can see (normalization failure, unnormalized resampling
 *    input) are written, first-error-wins, to a device int32 `status`
 *    (smc_wstate.status for the weight calls) and surface at the caller's next
 *    synchronization point -- the device analogue of SPEC.md:45/:137/:434.
 *  - Particle counts are int64 at the boundary; kernels support N < 2^31.
 *  - Threading: calls on distinct streams with distinct buffers are
 *    independent (rng.py:175-177 single-user-per-stream rule).
 */
#ifndef SMC_ABI_H
#define SMC_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMC_ABI_VERSION 3

#define SMC_OK 0
#define SMC_EINVAL -1         /* invalid argument                                   */
#define SMC_EUNNORMALIZED -2  /* resample input not normalized        */
#define SMC_ENORMALIZE -3     /* all -inf / NaN weights      */
#define SMC_EUNIFORMS -4      /* fewer explicit uniforms than the scheme draws      */
#define SMC_ECOUNTS -5        /* counts do not sum to N               */
#define SMC_ECUDA -6          /* CUDA launch / runtime error                        */
#define SMC_EWORKSPACE -7     /* workspace too small                                */

int smc_abi_version(void);
/* Copies the last host-side error message of the calling thread. */
int smc_last_error(char *buf, size_t len);
/* Kernels this library has launched in the process so far (every entry point's launches,
 * NVRTC user kernels included).  No reference counterpart: instrumentation for the bench's
 * `gpu_launches` (how many of the library's kernels ran in a timed region). */
int smc_launch_count(uint64_t *out);
/* Host-orchestration helper of a CUDA-graph-captured sampler loop (no reference counterpart:
 * the reference has no device history): hist[(*t - 1) * ncols + c] = row_prev[c], then
 * *t += 1, then obs_out[0..1] = obs[2 * *t .. +1] while *t < nobs -- the per-step history /
 * cursor / observation bookkeeping as ONE launch (t, obs_out, hist: device). */
int smc_graph_advance(const double *obs, int64_t nobs, double *obs_out, const double *row_prev, double *hist,
                      int64_t ncols, int64_t *t, void *stream);
/* Checked builds (-DSMC_CHECKED=1) count violated index guards in the kernels instead of
 * trapping; this returns their number and the first failing source line (1 = a checked
 * build, 0 = a production build, whose count is always 0).  Test infrastructure. */
int smc_check_failures(uint64_t *fails, uint64_t *first_line, char *file, size_t file_len);

/* ------------------------------------------------------------------------ */
/* RNG -- replaces pkg/src/smckit/rng.py                                     */
/* ------------------------------------------------------------------------ */
enum { SMC_DRAW_U01 = 0, SMC_DRAW_NORMAL = 1, SMC_DRAW_GAMMA = 2 };

/* Raw Philox4x32-10 blocks: out4[4i..4i+3] = philox(ctr4[4i..4i+3], key(seed)).
 * Replaces rng.py:59-72 (_philox_block); the KAT hook. */
int smc_philox_blocks(const uint32_t *ctr4, int64_t n, uint64_t seed, uint32_t *out4, void *stream);

/* n consecutive draws from ONE stream, advancing ctrs[stream_index] on device.
 * normal: out = mean + scale*z; gamma: out = scale*g(shape); u01: out = u.
 * Replaces rng.py:120-135 (fill_u01/fill_std_normal/fill_std_gamma) and
 * RngStream.uniform01/normal/gamma(n) (rng.py:186-215).  u01/normal draws are
 * computed in parallel (draw k uses counters c0+k / c0+2k, c0+2k+1); gamma is
 * sequential on one thread because its draw count is data dependent. */
int smc_rng_fill(int kind, uint64_t seed, uint64_t stream_index, uint64_t *ctrs, double shape,
                 double mean, double scale, double *out, int64_t n, void *stream);

/* One draw from each stream first..first+n-1 (the per-particle kernel pattern,
 * rng.py:75-117 called once per particle), advancing each counter. */
int smc_rng_draw_streams(int kind, uint64_t seed, uint64_t first_stream, int64_t n, uint64_t *ctrs,
                         double shape, double mean, double scale, double *out, void *stream);

/* ------------------------------------------------------------------------ */
/* Weights -- replaces smckit.weights.WeightSet             */
/* ------------------------------------------------------------------------ */
/* Device-resident weight state.  The log-weight vector is stored RAW
 * (lw_raw); the normalized log-weight is (lw_raw[i] - max_raw) - log_sum,
 * the oracle's max-shift + log-sum-exp order, or -log(N) for
 * every i when `equal` is set (set_equal_weight never touches the vector;
 * it sets max_raw = 0, log_sum = log N). */
typedef struct smc_wstate {
    double lse;        /* log sum_i exp(lw_raw_i)                               */
    double ess;        /* 1 / sum_i W_i^2                         */
    double ess_over_n; /* ess / N                                               */
    double nc_inc;     /* log sum_i W_{t-1,i} exp(incw_i) of the last ADD_LOG   */
    double log_zconst; /* running NormalizingConstant         */
    double max_raw;    /* max_i lw_raw_i                                        */
    double log_sum;    /* log sum_i exp(lw_raw_i - max_raw); lse = max + this   */
    double w_equal;    /* 1/N after set_equal_weight (N global when sharded)    */
    int32_t equal;     /* 1 after set_equal_weight                              */
    int32_t status;    /* sticky device error (SMC_E*), 0 when healthy          */
    int32_t resample;  /* decision of the last smc_ess_decide     */
    int32_t err_index; /* first failing particle of `status`, as INT32_MAX - i  */
    uint32_t lse_ticket; /* blocks of the running lse reduction that finished (the   */
    uint32_t reserved;   /* last one combines); 0 between calls -- create the record  */
                         /* zeroed                                                    */
} smc_wstate;

/* Every `int32_t *status` argument of this ABI points at an smc_status record (the
 * smc_wstate's status / resample / err_index words are one): the sticky error code,
 * then -- 8 bytes on -- the FIRST (lowest-index) failing particle, stored as
 * INT32_MAX - index so concurrent kernels keep the minimum with an atomic max; 0 = no
 * particle named ("first failing particle index reported"). */
typedef struct smc_status {
    int32_t code;
    int32_t reserved;
    int32_t first_index; /* INT32_MAX - index, 0 = none */
} smc_status;

enum { SMC_W_SET_LOG = 0, SMC_W_ADD_LOG = 1, SMC_W_SET_LIN = 2, SMC_W_MUL_LIN = 3, SMC_W_EQUAL = 4 };
enum { SMC_READ_LOG_WEIGHT = 0, SMC_READ_WEIGHT = 1 };

size_t smc_weights_workspace_bytes(int64_t n);
/* set_log_weight / add_log_weight / set_weight / mul_weight / set_equal_weight
 * (SPEC.md:31-69).  `values` is the new log-weight, log increment, weight or
 * factor vector (unused for EQUAL).  One pass over N plus a one-block
 * finalize; ADD_LOG also produces nc_inc and adds it to
 * log_zconst when `accumulate_nc` is set; SET_LOG with `accumulate_nc` starts
 * log_zconst at log (1/N) sum_i exp(values_i) (first weighting of an
 * equally weighted prior sample, e.g. the PF's init). */
int smc_weights_update(int mode, double *lw_raw, const double *values, int64_t n, smc_wstate *ws_state,
                       int accumulate_nc, void *ws, size_t ws_bytes, void *stream);
/* set_equal_weight gated by a device flag (skipped when
 * gate != NULL and *gate == 0): the post-resample reset of the sampler loop. */
int smc_weights_set_equal(smc_wstate *ws_state, int64_t n, const int32_t *gate, void *stream);
/* Multi-GPU normalization: combine G shard partials (SMC_PARTIAL_STRIDE
 * doubles each: max, sum e, sum e^2, monitor0, monitor1, pad) in rank order, so
 * every rank holds bit-identical global weight state; n_total is the global
 * particle count; monitor_out (2 doubles, may be NULL) gets the summed monitor. */
#define SMC_PARTIAL_STRIDE 8
int smc_weights_combine(const double *partials, int G, smc_wstate *ws_state, int64_t n_total, int mode,
                        int accumulate_nc, double *monitor_out, void *stream);
/* read_log_weight / read_weight: the normalized log-weight or its exp */
int smc_weights_read(int what, const double *lw_raw, const smc_wstate *ws_state, int64_t n, double *out,
                     void *stream);
/* ESS trigger: resample iff
 * threshold >= 1, or threshold > 0 and ess/N < threshold.  Writes
 * ws_state->resample; when hist_row != NULL also hist_row[0] = ess/N and
 * hist_row[1] = decision (the history record). */
int smc_ess_decide(smc_wstate *ws_state, int64_t n, double threshold, double *hist_row, void *stream);

/* Weighted sums out[j] = sum_i W_i * vals[i*ld + j], j < m  (monitor AW,
 * SPEC.md:320-326 / PAPER.md:574-586; path U_t).  W comes
 * from (lw_raw, ws_state).  Two passes: per-block partials, then a
 * fixed-order combine, so the result is run-to-run deterministic. */
size_t smc_weighted_reduce_workspace_bytes(int64_t n, int64_t m);
int smc_weighted_reduce(const double *vals, int64_t ld, int64_t m, const double *lw_raw,
                        const smc_wstate *ws_state, int64_t n, double *out, void *ws, size_t ws_bytes,
                        void *stream);

/* ------------------------------------------------------------------------ */
/* Resampling -- replaces smckit.resample                  */
/* ------------------------------------------------------------------------ */
enum {
    SMC_MULTINOMIAL = 0, SMC_RESIDUAL = 1, SMC_STRATIFIED = 2, SMC_SYSTEMATIC = 3,
    SMC_RESIDUAL_STRATIFIED = 4, SMC_RESIDUAL_SYSTEMATIC = 5
};

size_t smc_resample_workspace_bytes(int64_t n);

/* resample_<scheme>(W, stream) -> counts, + replication_to_parents, + the
 * value collection's copy, under the pinned
 * integer CDF contract.  Weights come from `w` (normalized W) or,
 * when w == NULL, from (lw_raw, ws_state) as W_i = exp(normalized lw_i).
 * Uniforms come from `u` (device, n_u of them) or, when u == NULL, from
 * stream `stream_index` of key(seed) starting at *ctr, which is advanced on
 * the device by the number of draws.  m_out is the number of
 * offspring (== n for a sampler; counts-only otherwise).  Outputs that are
 * NULL are skipped.  When rows != NULL every zero-count row j is overwritten
 * in place by row parents[j] (row_bytes each, 8-byte multiple) -- safe because
 * copy sources (count >= 2) and destinations (count 0) are disjoint.  When
 * gate != NULL and *gate == 0 every kernel returns immediately (device-side
 * ESS decision, no host sync).  Errors go to *status. */
int smc_resample(int scheme, const double *w, const double *lw_raw, const smc_wstate *ws_state, int64_t n,
                 int64_t m_out, uint64_t seed, uint64_t stream_index, uint64_t *ctr, const double *u,
                 int64_t n_u, int32_t *counts, int32_t *parents, void *rows, int64_t row_bytes,
                 const int32_t *gate, int32_t *status, void *ws, size_t ws_bytes, void *stream);

/* Test hook: SMC_DEBUG_FORCE_EXACT_F = 1 makes the stratified/systematic count
 * kernel always take its exact 128-bit path instead of the fp64 fast path
 * with guard band (the two are bit-identical by construction; tests check). */
/* SMC_DEBUG_MOVE_WS = 0 / 1 selects the PF move kernel: the single-role k_pf_move or the
 * warp-specialized k_pf_move_ws (Philox producer warps, Box-Muller consumer warps); the two
 * are bit-identical (tests/test_gpu_weights_pf.py). */
#define SMC_DEBUG_MOVE_WS 2
#define SMC_DEBUG_FORCE_EXACT_F 1
int smc_debug_set(int key, int value);

/* Sharded resampling over G GPUs (this shard holds particles [base, base+n)
 * of n_total; weights normalized globally, e.g. by smc_weights_combine).  The
 * counts and the global parent pairing are bit-identical to one GPU:
 *  1. smc_resample_shard_totals -> totals_out[4] = {T lo, T hi, sum f, T'};
 *     the host allgathers them into totals_all[G*4];
 *  2. smc_resample_shard_counts -> counts of the local particles (global CDF
 *     offset = exact integer prefix of the shards before), the local rank scan,
 *     zsp_out[4] = {zero slots Z, surplus children S, surplus parents P, active};
 *     the host allgathers zsp and plans the exchange: global zero rank r pairs
 *     with global surplus rank r; shard g owns zero ranks [Zoff_g, Zoff_g+Z_g)
 *     and surplus ranks [Soff_g, Soff_g+S_g);
 *  3. smc_resample_shard_pack -> rows of the local surplus children with local
 *     surplus ranks [ranges[2r], ranges[2r] + ranges[2r+1]) (host array, K <= 64),
 *     back to back, for ncclSend;
 *  4. smc_resample_shard_assign -> the local parent map; zero slots paired
 *     with a remote surplus child copy their row from `recv` (rows ordered by
 *     global rank, the shard's own range [soff, soff+s_self) excluded) and
 *     keep parents[j] = j; local pairs get the local parent index. */
int smc_resample_shard_totals(int scheme, const double *w, const double *lw_raw, const smc_wstate *ws_state,
                              int64_t n, int64_t n_total, int64_t m_total, const double *u, int64_t n_u,
                              const int32_t *gate, int32_t *status, void *ws, size_t ws_bytes, uint64_t *totals_out,
                              void *stream);
int smc_resample_shard_counts(int scheme, const double *w, const double *lw_raw, const smc_wstate *ws_state,
                              int64_t n, int64_t n_total, int64_t m_total, int G, int rank,
                              const uint64_t *totals_all, uint64_t seed, uint64_t stream_index, uint64_t *ctr,
                              const double *u, int64_t n_u, int32_t *counts, const int32_t *gate, int32_t *status,
                              void *ws, size_t ws_bytes, uint32_t *zsp_out, void *stream);
int smc_resample_shard_pack(const void *rows, int64_t row_bytes, int64_t n, const int64_t *ranges, int K,
                            void *sendbuf, void *ws, size_t ws_bytes, void *stream);
int smc_resample_shard_assign(const int32_t *counts, int64_t n, int64_t zoff, int64_t soff, int64_t s_self,
                              const void *recv, void *rows, int64_t row_bytes, int32_t *parents, void *ws,
                              size_t ws_bytes, void *stream);

/* The same assignment with the cross-shard rows read straight from the other ranks' memory
 * (CUDA-IPC mappings, P2P loads over NVLink/NVSwitch) instead of a packed send/receive:
 * zsp_all = the allgathered smc_resample_shard_counts outputs (G x {Z, S, P, active}, device),
 * peer_ws[r] / peer_rows[r] = rank r's resample workspace and current state buffer (host
 * arrays of G device pointers; the own rank's entries are its own buffers).  Every offset
 * comes from zsp_all on the device: no host plan and no host synchronization per step.
 * The allgather that delivered zsp_all orders this call after every peer's counts pass.
 * Replaces the row-migration step of PAPER.md:1993-2059 (vSMC MPI module). */
int smc_resample_shard_assign_p2p(const uint32_t *zsp_all, int G, int rank, const void *const *peer_ws,
                                  const void *const *peer_rows, int64_t n, void *rows, int64_t row_bytes,
                                  int32_t *parents, int32_t *status, void *ws, size_t ws_bytes, void *stream);

/* replication_to_parents(counts) from a device counts vector. */
int smc_replication_to_parents(const int32_t *counts, int64_t n, int32_t *parents, int32_t *status, void *ws,
                               size_t ws_bytes, void *stream);

/* StateMatrix.copy_particles(parents), simultaneous: dst row
 * j <- src row parents[j]; dst != src (out of place). */
int smc_gather_rows(void *dst, const void *src, int64_t row_bytes, const int32_t *parents, int64_t n,
                    void *stream);
/* In-place variant for a ParentVector (copy_from[j] == j whenever j survives):
 * copies only rows with parents[j] != j. */
int smc_copy_rows_inplace(void *rows, int64_t row_bytes, const int32_t *parents, int64_t n,
                          const int32_t *gate, void *stream);

/* ------------------------------------------------------------------------ */
/* example-pf kernels -- replace cv_init / cv_move / cv_monitor              */
/*               */
/* ------------------------------------------------------------------------ */
size_t smc_pf_workspace_bytes(int64_t n);
/* X (n x 4 row-major f64) ~ prior from streams 0..n-1 (draw order x,y,vx,vy),
 * llh at obs_t = (x_obs, y_obs) (device, 2 doubles) -> set_log_weight; the
 * state's log_zconst restarts at log (1/N) sum exp(llh). */
int smc_pf_init(double *x, double *lw_raw, int64_t n, uint64_t stream_base, uint64_t seed, uint64_t *ctrs,
                const double *obs_t, smc_wstate *ws_state, double *partial_out, void *ws, size_t ws_bytes,
                void *stream);
/* Sharded systems (particles [stream_base, stream_base + n) of N_total on
 * this GPU): the Philox stream of local particle i is stream_base + i, and
 * with partial_out != NULL the normalization is NOT applied locally -- the
 * shard's {max, sum e, sum e^2, mon0, mon1} (SMC_PARTIAL_STRIDE doubles) is
 * written there for the ranks to allgather and smc_weights_combine. */
/* cv_move on every particle + incw = llh(t) -> add_log_weight(incw) fused in
 * one pass over the state; log_zconst += log sum W_{t-1} exp(incw).
 * incw_out may be NULL. */
int smc_pf_move(const double *x_in, double *x, const int32_t *parents, const int32_t *gate, double *lw_raw,
                int64_t n, uint64_t stream_base, int64_t n_total, uint64_t seed, uint64_t *ctrs,
                const double *obs_t, smc_wstate *ws_state, double *incw_out, double *monitor_prev,
                double *partial_out, void *ws, size_t ws_bytes, void *stream);
/* x_in / parents / gate fold the previous resample's copy into the move: row i
 * is read from x_in[parents[i]] (x_in[i] when parents is NULL or *gate == 0)
 * and written to x[i] -- copy_particles' simultaneous semantics
 * by double buffering, so the resample never copies rows.  x_in == NULL means
 * x_in = x (in place, parents must then be NULL). */
/* monitor_prev (device, 2 doubles, may be NULL): receives the "pos" monitor
 * sum_i W_i (x_i, y_i) of the state the move CONSUMES -- the previous
 * iteration's estimate -- reduced from registers the move
 * already holds, so the monitor costs no extra pass over the state. */
/* smc_pf_move when every stream 0..n-1 is known to sit at the same draw count
 * ctr (the host's RngStreamSet tracks this; SPEC.md:396 own-slot streams):
 * same results bit for bit, but the counter array is neither read nor written
 * (the host records the advanced count, ctr + 8) and the Philox blocks share
 * their stream-only products.  SMC_EINVAL if lo32(ctr) + 15 would carry or
 * stream_base + n > 2^32. */
int smc_pf_move_uniform(const double *x_in, double *x, const int32_t *parents, const int32_t *gate,
                        double *lw_raw, int64_t n, uint64_t stream_base, int64_t n_total, uint64_t seed,
                        uint64_t ctr, const double *obs_t, smc_wstate *ws_state, double *incw_out,
                        double *monitor_prev, double *partial_out, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* example-gmm kernels -- replace gmm_init / gmm_move_smc / gmm_move_{mu,   */
/* lambda,weight} / gmm_path          */
/* ------------------------------------------------------------------------ */
/* State: n x SMC_GMM_ROW f64 row-major per particle: mu[4], lambda[4],
 * omega[4], log_prior, log_likelihood, 2 pad; components j < r (1 <= r <=
 * SMC_GMM_MAX_R) are live, the rest stay 0.  data: the observations (device,
 * nd <= SMC_GMM_MAX_DATA).  hyper (host, 6 doubles): xi, kappa, nu, chi, rho,
 * lambda_known of mu ~ N(xi, 1/kappa), lambda ~ Gamma(nu, scale chi), omega ~
 * Dirichlet(rho); lambda_known > 0 fixes every lambda_j at that precision (no
 * Gamma term, no lambda move: the conjugate-oracle model of SPEC.md:586-587). */
#define SMC_GMM_ROW 16
#define SMC_GMM_MAX_R 4
#define SMC_GMM_MAX_DATA 4096
/* gmm_init: per component mu, lambda (unless known), Gamma(1,1)
 * weight (in that order, from stream stream_base + i); weights normalized; caches set. */
int smc_gmm_init(double *x, int64_t n, int r, uint64_t stream_base, uint64_t seed, uint64_t *ctrs,
                 const double *data, int nd, const double *hyper, void *stream);
/* Recompute the log_prior / log_likelihood caches of every row. */
int smc_gmm_eval(double *x, int64_t n, int r, const double *data, int nd, const double *hyper, void *stream);
size_t smc_gmm_workspace_bytes(int64_t n);
/* gmm_move_smc's weight update: incw_i = dalpha * llh_i,
 * log_zconst += log sum W_{t-1} exp(incw), add_log_weight(incw) -- fused. */
int smc_gmm_reweight(const double *x, double *lw_raw, int64_t n, double dalpha, smc_wstate *ws_state,
                     double *partial_out, void *ws, size_t ws_bytes, void *stream);
/* gmm_move_mu (block 0), _lambda (1, log scale), _weight (2, r-1 logits) random-walk
 * Metropolis at temperature alpha with proposal scale sd:
 * accept iff log U < p_new - p_old (+ Jacobian); *accepted += #accepted. */
int smc_gmm_mh(int block, double *x, int64_t n, int r, uint64_t stream_base, uint64_t seed, uint64_t *ctrs,
               const double *data, int nd, const double *hyper, double alpha, double sd,
               unsigned long long *accepted, void *stream);

/* ------------------------------------------------------------------------ */
/* user particle kernels, compiled at run time -- replaces the per-particle  */
/* `kernel(iter, SingleParticleView) -> int` / MoveAdapter / monitor and    */
/* path evaluators      */
/* ------------------------------------------------------------------------ */
/* source: CUDA C++ that includes "smc_user.cuh" (pass -I<csrc dir> in
 * options) and ends with SMC_USER_MOVE(fn) or SMC_USER_EVAL(fn).  NVRTC
 * compiles it for sm_100a (--fmad=false); libnvrtc / libcuda are loaded on
 * first use.  log (may be NULL) receives the compiler log.  The module handle
 * is freed with smc_user_free. */
#define SMC_USER_MOVE 1
#define SMC_USER_EVAL 2
int smc_user_compile(const char *source, const char *const *options, int n_options, void **module_out, char *log,
                     size_t log_bytes);
int smc_user_kind(const void *module);
int smc_user_free(void *module);
/* One thread per particle: fn(Particle&, iter, params) with the particle's row
 * of x (n x dim, row- or column-major), its stream stream_base + i (counter
 * ctrs[i], written back), scratch row i (n x sdim); *accepted += sum of the
 * returned ints (exact). */
int smc_user_launch_move(void *module, uint64_t iter, double *x, int64_t n, int dim, int col_major,
                         uint64_t stream_base, uint64_t seed, uint64_t *ctrs, double *scratch, int sdim,
                         const double *params, unsigned long long *accepted, void *stream);
/* fn(const Particle&, iter, params, out + i*m): m values per particle (a monitor's
 * h_1..h_m, res[i*dim + j] of PAPER.md:574-586, or a path integrand with m = 1). */
int smc_user_launch_eval(void *module, uint64_t iter, const double *x, int64_t n, int dim, int col_major,
                         const double *params, double *out, int m, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SMC_ABI_H */
