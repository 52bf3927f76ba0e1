// smc_pf.cu -- the paper's particle filter kernels:
// cv_init / cv_move fused with the weight update and the one-pass log-sum-exp
// / ESS partials, so a PF step reads and writes the state exactly once.
//
// State: X is N x 4 f64 row-major, one 32-byte row per particle,
// moved with one 256-bit load and one 256-bit store per thread.
// Per particle-step HBM traffic: X 32 R + 32 W, lw 8 R (skipped after a
// resample: equal weights) + 8 W  =  80 B, + counter 8 R + 8 W when the
// streams are not all at one count (smc_pf_move vs smc_pf_move_uniform).
#include "smc_weights.cuh"

using namespace smc;

namespace {

#ifndef PF_PB
#define PF_PB 128  // threads per PF block (same-box A/B: 128 x 8 blocks/SM 2 % faster than 256 x 4)
#endif
constexpr int PB = PF_PB;
#ifndef PF_MIN_BLOCKS
#define PF_MIN_BLOCKS 8
#endif
#ifndef PF_PPT
#define PF_PPT 8  // particles per thread in the move kernel (same-box A/B: 8 > 4 by ~1 %)
#endif
#ifndef PF_UNROLL
#define PF_UNROLL 1  // particles of a thread interleaved by the compiler (ILP vs registers)
#endif
constexpr int kPfUnroll = PF_UNROLL;
#ifndef PF_SWP
#define PF_SWP 0  // software-pipelined move body (next particle's draws beside this one's Box-Muller)
#endif
template <bool B>
struct BoolTag {
    static constexpr bool value = B;
};
constexpr int MB = PB * PF_PPT;  // particles per move block
#ifndef SMC_MOVE_WS_DEFAULT
#define SMC_MOVE_WS_DEFAULT 0  // the single-role move; the warp-specialized k_pf_move_ws measured slower (profiles/r2_move_ws_ab.txt)
#endif

struct PfConst {
    double sd_pos0, sd_vel0;  // init: 2, 1
    double sd_pos, sd_vel;    // move: sqrt(.02), sqrt(.001)
    double delta;             // 0.1
};

// PAPER.md:1181-1191 / SPEC.md:464-472 (scale 10, nu 10).  log(1 + a) + log(1 + b)
// is taken as ONE log of the product (one fewer fp64 log per particle-step;
// the two-log form only if the product overflows): agrees with the reference's
// two logs to an absolute 2e-16 in the log-weight.
// the reference's two logs, for the (never seen in practice) overflowing product: out of line so
// the libm fallback's code and registers stay out of the move loop
__device__ __noinline__ double log_sum_cold(double ax, double ay)
{
    return smc_fm::log(ax) + smc_fm::log(ay);
}

SMC_DEV double cv_llh(double xp, double yp, double xo, double yo, const smc_fm::LogEntry *logtab = nullptr)
{
    const double scale = 10;
    const double nu = 10;
    const double rx = scale * (xp - xo);
    const double ry = scale * (yp - yo);
    const double ax = 1 + smc_fm::div10(rx * rx);  // 1 + rx^2 / nu (nu = 10)
    const double ay = 1 + smc_fm::div10(ry * ry);
    const double p = ax * ay;
    const double s = p < INFINITY ? smc_fm::log_core(p, logtab) : log_sum_cold(ax, ay);  // p >= 1
    return -0.5 * (nu + 1) * s;
}

SMC_DEV void ld_row(const double *p, double &a, double &b, double &c, double &d)
{
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
SMC_DEV void st_row(double *p, double a, double b, double c, double d)
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__global__ void __launch_bounds__(PB) k_pf_init(double *__restrict__ x, double *__restrict__ lw_raw, int64_t n,
                                                uint64_t sbase, const KeySched key, uint64_t *__restrict__ ctrs,
                                                const double *__restrict__ obs,
                                                PfConst k, smc_wstate *st, LsePartial *__restrict__ parts)
{
    SMC_PDL_WAIT();
    const int64_t i = (int64_t)blockIdx.x * PB + threadIdx.x;
    double v = -INFINITY;
    if (i < n) {
        const uint64_t c = ctrs[i], si = sbase + (uint64_t)i;  // global stream index of a sharded system
        // draw order x_pos, y_pos, x_vel, y_vel; normal = mean + sd*z (rng.py:201)
        double z[4];
        normals_at(c, si, key, z);
        const double r0 = 0.0 + k.sd_pos0 * z[0];
        const double r1 = 0.0 + k.sd_pos0 * z[1];
        const double r2 = 0.0 + k.sd_vel0 * z[2];
        const double r3 = 0.0 + k.sd_vel0 * z[3];
        ctrs[i] = c + 8;
        st_row(x + 4 * i, r0, r1, r2, r3);
        v = cv_llh(r0, r1, obs[0], obs[1]);
        if (isnan(v)) { raise_status_at(&st->status, SMC_ENORMALIZE, (int64_t)si); v = -INFINITY; }
        lw_raw[i] = v;  // set_log_weight(llh)
    }
    LsePartial p = block_lse_partial<PB>(v);
    if (threadIdx.x == 0) parts[blockIdx.x] = p;
}

// MON: also reduce the "pos" monitor of the INCOMING state, sum_i W_{t-1,i} (x_i, y_i) -- the
// previous iteration's estimate (evaluated after its resample) --
// from the registers the move already holds: the monitor costs no extra HBM pass.
// GATHER: the previous resample's copy is folded in -- row i is read from
// x_in[parents[i]] (when the device gate says the resample ran) and written to
// x_out[i], a second buffer: the "simultaneous" copy of SPEC.md:343 for free.
// PPT particles per thread (striped: particle base + k*PB, k < PPT, so every
// warp access stays coalesced): the block's lse/ESS and monitor reductions are
// paid once per PPT particles.  The body runs in a non-unrolled loop (code size:
// the move is ~2.7k SASS); each particle's new log-weight parks in shared memory
// until the block max is known.
// The fast-math tables (log 8 KB, cos 320 B, exp 2 KB) staged in shared memory once per
// block: 32-bit shared addressing instead of a 64-bit global address (constant-bank base +
// IMAD.WIDE on the FMA pipe, which the Philox multiplies saturate) per lookup.
struct __align__(16) PfTabs {
    smc_fm::LogEntry log[512];
    smc_fm::ExpEntry exp[128];
    smc_fm::CosPoly cos[4];
};
// The tables are staged in two halves: every 16-byte piece loaded into registers
// first (tab_load), the shared stores and the barrier only after the block's parent indices
// and first prefetches are in flight too (tab_store) -- one memory round trip at block start
// instead of two.
static_assert(sizeof(smc_fm::LogEntry) == 16 && sizeof(smc_fm::ExpEntry) == 16 && sizeof(PfTabs::cos) == 320,
              "table layout");
static_assert(PB >= 128 && 512 % PB == 0, "one pass of 16-byte pieces per table");
struct TabRegs {
    double2 log[512 / PB], exp, cos;
};
SMC_DEV void tab_load(TabRegs &r)
{
    const double2 *lg = reinterpret_cast<const double2 *>(smc_fm::kLogTab);
#pragma unroll
    for (int k = 0; k < 512 / PB; ++k) r.log[k] = __ldg(lg + threadIdx.x + k * PB);
    if (threadIdx.x < 128) r.exp = __ldg(reinterpret_cast<const double2 *>(smc_fm::kExpTab) + threadIdx.x);
    if (threadIdx.x < 20) r.cos = __ldg(reinterpret_cast<const double2 *>(smc_fm::kCosPoly) + threadIdx.x);
}
SMC_DEV void tab_store(PfTabs &t, const TabRegs &r)
{
#pragma unroll
    for (int k = 0; k < 512 / PB; ++k) reinterpret_cast<double2 *>(t.log)[threadIdx.x + k * PB] = r.log[k];
    if (threadIdx.x < 128) reinterpret_cast<double2 *>(t.exp)[threadIdx.x] = r.exp;
    if (threadIdx.x < 20) reinterpret_cast<double2 *>(t.cos)[threadIdx.x] = r.cos;
    __syncthreads();
}

// UC: every particle's stream at the same draw count ctr_u (no carry over its 8 draws; the
// host tracks this, rng.py): the counter array is neither read nor written (16 B per
// particle-step less traffic) and the Philox blocks use normals_uniform (16 multiplies per
// draw instead of 20).
template <bool MON, int PPT, bool UC>
__global__ void __launch_bounds__(PB, PF_MIN_BLOCKS) k_pf_move(const double *x_in, double *x_out,
                                                   const int32_t *__restrict__ parents, const int32_t *gate,
                                                   double *__restrict__ lw_raw, int64_t n, uint64_t sbase,
                                                   double w_equal, const KeySched key, uint64_t *__restrict__ ctrs, const UniformCtr ctr_u,
                                                   const double *__restrict__ obs, PfConst k, smc_wstate *st, double *__restrict__ incw_out,
                                                   LsePartial *__restrict__ parts, double2 *__restrict__ mon_parts)
{
    __shared__ PfTabs tabs;
    TabRegs tr;
    tab_load(tr);  // constant data: requested before the dependency wait
    SMC_PDL_WAIT();
    __shared__ double s_v[PPT][PB];
    const int64_t base = (int64_t)blockIdx.x * (PB * PPT) + threadIdx.x;
    double h0 = 0.0, h1 = 0.0;
    const NormLw nl = norm_of(st);
    const bool gathered = parents && (gate == nullptr || *gate != 0);
    const double xo = obs[0], yo = obs[1];
    // software prefetch: the next particle's counter and old log-weight are requested before
    // this particle's normals, so their latency hides behind the Philox work
    // the block's parent indices (PPT x PB, 4 bytes each) staged in shared memory up front with
    // coalesced loads: each particle's gathered row load then needs no dependent global load
    __shared__ int32_t s_src[PPT][PB];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int64_t i = base + (int64_t)q * PB;
        s_src[q][threadIdx.x] = gathered && i < n ? __ldg(parents + i) : (int32_t)i;
    }
    uint64_t c_nx = 0;
    double lw_nx = 0.0;
    if (base < n) {
        if (!UC) c_nx = ctrs[base];
        if (nl.needs_raw()) lw_nx = lw_raw[base];
    }
    tab_store(tabs, tr);
#if PF_SWP
    // Software-pipelined body (uniform counts, every particle of the thread in range): the
    // Philox draws of particle q + 1 are computed in the same basic block as particle q's
    // Box-Muller transforms, so each warp's instruction stream mixes IMAD.WIDE / LOP3 (FMA and
    // ALU pipes) with the fp64 work instead of alternating a Philox phase and an fp64 phase.
    // Same arithmetic per particle: bit-identical to the loop below.
    if (UC && PPT > 1 && base + (int64_t)(PPT - 1) * PB < n) {
        double2 a[4];
        {
            uint64_t m[8];
            draws_uniform<8>(ctr_u, sbase + (uint64_t)base, key, m);
#pragma unroll
            for (int j = 0; j < 4; ++j) a[j] = box_muller_args(m[2 * j], m[2 * j + 1]);
        }
        auto body = [&](int q, auto next) {
            constexpr bool NEXT = decltype(next)::value;
            const int64_t i = base + (int64_t)q * PB;
            const int64_t src = s_src[q][threadIdx.x];
            const double lw_prev = lw_nx;
            if (NEXT && nl.needs_raw()) lw_nx = lw_raw[i + PB];
            const double prev = nl(lw_prev);
            double x0, x1, x2, x3;
            SMC_CHECK(src >= 0 && src < n);
            ld_row(x_in + 4 * src, x0, x1, x2, x3);
            const uint64_t si = sbase + (uint64_t)i;
            double2 an[4];
            if constexpr (NEXT) {
                uint64_t m[8];
                draws_uniform<8>(ctr_u, si + PB, key, m);
#pragma unroll
                for (int j = 0; j < 4; ++j) an[j] = box_muller_args(m[2 * j], m[2 * j + 1]);
            }
            double z[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) z[j] = box_muller_from(a[j], FmTabs{tabs.log, tabs.cos});
            if constexpr (NEXT) {
#pragma unroll
                for (int j = 0; j < 4; ++j) a[j] = an[j];
            }
            if (MON) {
                const double w = nl.eq ? w_equal : smc_fm::exp(prev, tabs.exp);
                h0 += w * x0;
                h1 += w * x1;
            }
            x0 = x0 + ((0.0 + k.sd_pos * z[0]) + k.delta * x2);
            x1 = x1 + ((0.0 + k.sd_pos * z[1]) + k.delta * x3);
            x2 = x2 + (0.0 + k.sd_vel * z[2]);
            x3 = x3 + (0.0 + k.sd_vel * z[3]);
            st_row(x_out + 4 * i, x0, x1, x2, x3);
            const double incw = cv_llh(x0, x1, xo, yo, tabs.log);
            if (incw_out) incw_out[i] = incw;
            double v = prev + incw;
            if (isnan(v) || v == INFINITY) { raise_status_at(&st->status, SMC_ENORMALIZE, (int64_t)si); v = -INFINITY; }
            lw_raw[i] = v;
            s_v[q][threadIdx.x] = v;
        };
#pragma unroll 1
        for (int q = 0; q < PPT - 1; ++q) body(q, BoolTag<true>{});
        body(PPT - 1, BoolTag<false>{});
    } else
#endif
#pragma unroll kPfUnroll
    for (int q = 0; q < PPT; ++q) {
        const int64_t i = base + (int64_t)q * PB;
        double v = -INFINITY;
        const uint64_t c = c_nx;
        const int64_t src = s_src[q][threadIdx.x];
        const double lw_prev = lw_nx;
        if (q + 1 < PPT && i + PB < n) {
            if (!UC) c_nx = ctrs[i + PB];
            if (nl.needs_raw()) lw_nx = lw_raw[i + PB];
        }
        if (i < n) {
            const double prev = nl(lw_prev);  // normalized W_{t-1}; no read if equal
            double x0, x1, x2, x3;
            SMC_CHECK(src >= 0 && src < n);
            ld_row(x_in + 4 * src, x0, x1, x2, x3);
            const uint64_t si = sbase + (uint64_t)i;
            // PAPER.md:1310-1313, evaluation order pinned: x0 += (0 + sd*z) + delta*x2
            double z[4];
            if (UC)
                normals_uniform(ctr_u, si, key, z, FmTabs{tabs.log, tabs.cos});
            else
                normals_at(c, si, key, z, FmTabs{tabs.log, tabs.cos});  // the row load lands meanwhile
            if (MON) {
                const double w = nl.eq ? w_equal : smc_fm::exp(prev, tabs.exp);  // 1 / N_total after a resample
                h0 += w * x0;
                h1 += w * x1;
            }
            x0 = x0 + ((0.0 + k.sd_pos * z[0]) + k.delta * x2);
            x1 = x1 + ((0.0 + k.sd_pos * z[1]) + k.delta * x3);
            x2 = x2 + (0.0 + k.sd_vel * z[2]);
            x3 = x3 + (0.0 + k.sd_vel * z[3]);
            if (!UC) ctrs[i] = c + 8;
            st_row(x_out + 4 * i, x0, x1, x2, x3);
            const double incw = cv_llh(x0, x1, xo, yo, tabs.log);
            if (incw_out) incw_out[i] = incw;
            v = prev + incw;  // add_log_weight(incw)
            if (isnan(v) || v == INFINITY) { raise_status_at(&st->status, SMC_ENORMALIZE, (int64_t)si); v = -INFINITY; }
            lw_raw[i] = v;
        }
        s_v[q][threadIdx.x] = v;
    }
    SMC_PDL_TRIGGER();  // the lse combine's blocks may launch now (they wait for this grid)
    // block (max, sum e, sum e^2), e = exp(v - max): one pass over the parked values
    __shared__ double s_red[3][PB / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double tm = s_v[0][threadIdx.x];
#pragma unroll
    for (int q = 1; q < PPT; ++q) tm = fmax(tm, s_v[q][threadIdx.x]);
    tm = warp_max(tm);
    if (lane == 0) s_red[0][warp] = tm;
    __syncthreads();
    double bm = lane < PB / 32 ? s_red[0][lane] : -INFINITY;
    bm = warp_max(bm);  // every warp reduces the 8 warp maxima itself: no second barrier
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const double e = smc_fm::exp(s_v[q][threadIdx.x] - bm, tabs.exp);  // -inf -> 0
        s1 += e;
        s2 += e * e;
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (MON) {
        h0 = warp_sum(h0);
        h1 = warp_sum(h1);
    }
    __syncthreads();  // s_red[0] reads are done
    if (lane == 0) {
        s_red[1][warp] = s1;
        s_red[2][warp] = s2;
        if (MON) { s_v[0][warp] = h0; s_v[1 % PPT][PB / 32 + warp] = h1; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        LsePartial p{bm, 0.0, 0.0};
        double a = 0.0, b = 0.0;
        for (int w = 0; w < PB / 32; ++w) {
            p.s1 += s_red[1][w];
            p.s2 += s_red[2][w];
            if (MON) { a += s_v[0][w]; b += s_v[1 % PPT][PB / 32 + w]; }
        }
        parts[blockIdx.x] = p;
        if (MON) mon_parts[blockIdx.x] = make_double2(a, b);
    }
}

// ---------------------------------------------------------------------------------------------
// Warp-specialized move (same arithmetic, bit-identical results): a block of 8 warps, 4
// PRODUCER warps computing the Philox draws (IMAD.WIDE + LOP3: the FMA / ALU pipes) and 4
// CONSUMER warps doing Box-Muller, the move, the likelihood and the lse/ESS partials (the fp64
// pipe), so that at any moment the warps of a scheduler mix both instruction streams instead of
// every warp alternating between a Philox phase and an fp64 phase.  The draws of a stage (one
// particle per consumer thread) pass through a 2-slot shared-memory ring, [slot][draw][thread]
// (consecutive threads, consecutive words: conflict-free), handed over with named barriers:
// FULL (producers arrive, consumers wait) and EMPTY (consumers arrive, producers wait).
constexpr int WSC = 128;  // consumer threads
constexpr int WSP = 128;  // producer threads
constexpr int WST = WSC + WSP;
SMC_DEV void nbar_sync(int id, int count) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }
SMC_DEV void nbar_arrive(int id, int count) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory"); }
constexpr int WS_SLOTS = 3;  // ring slots: the producers may run up to 3 stages ahead (48 KB static shared)
enum { BAR_CONS = 1, BAR_FULL = 2, BAR_EMPTY = 2 + WS_SLOTS };  // FULL / EMPTY: one id per ring slot

template <bool MON, int PPT, bool UC>
__global__ void __launch_bounds__(WST, 4) k_pf_move_ws(const double *x_in, double *x_out,
                                                  const int32_t *__restrict__ parents, const int32_t *gate,
                                                  double *__restrict__ lw_raw, int64_t n, uint64_t sbase,
                                                  double w_equal, const KeySched key, uint64_t *__restrict__ ctrs, const UniformCtr ctr_u,
                                                  const double *__restrict__ obs, PfConst k, smc_wstate *st, double *__restrict__ incw_out,
                                                  LsePartial *__restrict__ parts, double2 *__restrict__ mon_parts)
{
    __shared__ PfTabs tabs;
    __shared__ double2 ring[WS_SLOTS][4][WSC];  // Box-Muller arguments (1 - u1, 2 pi u2) per normal
    __shared__ double s_v[PPT][WSC];
    __shared__ int32_t s_src[PPT][WSC];
    const int64_t blk = (int64_t)blockIdx.x * (WSC * PPT);
    if (threadIdx.x >= WSC) {  // ---------------- producers: the draws ----------------
        SMC_PDL_WAIT();
        const int p = threadIdx.x - WSC;
        for (int q = 0; q < PPT; ++q) {
            const int slot = q % WS_SLOTS;
            const int64_t i = blk + (int64_t)q * WSC + p;
            uint64_t m[8];
            if (i < n) {
                const uint64_t si = sbase + (uint64_t)i;
                if (UC) {
                    draws_uniform<8>(ctr_u, si, key, m);
                } else {
                    const uint64_t c = ctrs[i];
#pragma unroll
                    for (int j = 0; j < 8; ++j) m[j] = draw53(c + (uint64_t)j, si, key);
                    ctrs[i] = c + 8;
                }
            }
            double2 a[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) a[j] = box_muller_args(m[2 * j], m[2 * j + 1]);  // conversions here too
            if (q >= WS_SLOTS) nbar_sync(BAR_EMPTY + slot, WST);  // the consumers are done with this slot
            if (i < n) {
#pragma unroll
                for (int j = 0; j < 4; ++j) ring[slot][j][p] = a[j];  // 128-bit stores, conflict-free
            }
            nbar_arrive(BAR_FULL + slot, WST);
        }
        return;
    }
    // ---------------- consumers: Box-Muller, move, likelihood, weights ----------------
    TabRegs tr;
    tab_load(tr);  // constant data: requested before the dependency wait
    SMC_PDL_WAIT();
    const int64_t base = blk + threadIdx.x;
    double h0 = 0.0, h1 = 0.0;
    const NormLw nl = norm_of(st);
    const bool gathered = parents && (gate == nullptr || *gate != 0);
    const double xo = obs[0], yo = obs[1];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int64_t i = base + (int64_t)q * WSC;
        s_src[q][threadIdx.x] = gathered && i < n ? __ldg(parents + i) : (int32_t)i;
    }
    double lw_nx = 0.0;
    if (base < n && nl.needs_raw()) lw_nx = lw_raw[base];
#pragma unroll
    for (int k2 = 0; k2 < 512 / WSC; ++k2) reinterpret_cast<double2 *>(tabs.log)[threadIdx.x + k2 * WSC] = tr.log[k2];
    reinterpret_cast<double2 *>(tabs.exp)[threadIdx.x] = tr.exp;
    if (threadIdx.x < 20) reinterpret_cast<double2 *>(tabs.cos)[threadIdx.x] = tr.cos;
    nbar_sync(BAR_CONS, WSC);
#pragma unroll 1
    for (int q = 0; q < PPT; ++q) {
        const int slot = q % WS_SLOTS;
        const int64_t i = base + (int64_t)q * WSC;
        double v = -INFINITY;
        const int64_t src = s_src[q][threadIdx.x];
        const double lw_prev = lw_nx;
        if (q + 1 < PPT && i + WSC < n && nl.needs_raw()) lw_nx = lw_raw[i + WSC];
        double x0 = 0, x1 = 0, x2 = 0, x3 = 0;
        if (i < n) ld_row(x_in + 4 * src, x0, x1, x2, x3);  // requested before the wait for the draws
        nbar_sync(BAR_FULL + slot, WST);
        double2 a[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = ring[slot][j][threadIdx.x];
        if (q + WS_SLOTS < PPT) nbar_arrive(BAR_EMPTY + slot, WST);
        if (i < n) {
            const double prev = nl(lw_prev);
            double z[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) z[j] = box_muller_from(a[j], FmTabs{tabs.log, tabs.cos});
            if (MON) {
                const double w = nl.eq ? w_equal : smc_fm::exp(prev, tabs.exp);
                h0 += w * x0;
                h1 += w * x1;
            }
            x0 = x0 + ((0.0 + k.sd_pos * z[0]) + k.delta * x2);
            x1 = x1 + ((0.0 + k.sd_pos * z[1]) + k.delta * x3);
            x2 = x2 + (0.0 + k.sd_vel * z[2]);
            x3 = x3 + (0.0 + k.sd_vel * z[3]);
            st_row(x_out + 4 * i, x0, x1, x2, x3);
            const double incw = cv_llh(x0, x1, xo, yo, tabs.log);
            if (incw_out) incw_out[i] = incw;
            v = prev + incw;
            if (isnan(v) || v == INFINITY) {
                raise_status_at(&st->status, SMC_ENORMALIZE, (int64_t)(sbase + (uint64_t)i));
                v = -INFINITY;
            }
            lw_raw[i] = v;
        }
        s_v[q][threadIdx.x] = v;
    }
    SMC_PDL_TRIGGER();
    __shared__ double s_red[3][WSC / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double tm = s_v[0][threadIdx.x];
#pragma unroll
    for (int q = 1; q < PPT; ++q) tm = fmax(tm, s_v[q][threadIdx.x]);
    tm = warp_max(tm);
    if (lane == 0) s_red[0][warp] = tm;
    nbar_sync(BAR_CONS, WSC);
    double bm = lane < WSC / 32 ? s_red[0][lane] : -INFINITY;
    bm = warp_max(bm);
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const double e = smc_fm::exp(s_v[q][threadIdx.x] - bm, tabs.exp);
        s1 += e;
        s2 += e * e;
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (MON) {
        h0 = warp_sum(h0);
        h1 = warp_sum(h1);
    }
    nbar_sync(BAR_CONS, WSC);
    if (lane == 0) {
        s_red[1][warp] = s1;
        s_red[2][warp] = s2;
        if (MON) { s_v[0][warp] = h0; s_v[1 % PPT][WSC / 32 + warp] = h1; }
    }
    nbar_sync(BAR_CONS, WSC);
    if (threadIdx.x == 0) {
        LsePartial pp{bm, 0.0, 0.0};
        double a = 0.0, b = 0.0;
        for (int w = 0; w < WSC / 32; ++w) {
            pp.s1 += s_red[1][w];
            pp.s2 += s_red[2][w];
            if (MON) { a += s_v[0][w]; b += s_v[1 % PPT][WSC / 32 + w]; }
        }
        parts[blockIdx.x] = pp;
        if (MON) mon_parts[blockIdx.x] = make_double2(a, b);
    }
}

int h_move_ws = SMC_MOVE_WS_DEFAULT;  // which move kernel runs (smc_debug_set SMC_DEBUG_MOVE_WS)

PfConst pf_constants()
{
    PfConst k;
    k.sd_pos0 = 2;
    k.sd_vel0 = 1;
    k.sd_pos = sqrt(0.02);
    k.sd_vel = sqrt(0.001);
    k.delta = 0.1;
    return k;
}

}  // namespace

extern "C" size_t smc_pf_workspace_bytes(int64_t n)
{
    return (size_t)((n + PB - 1) / PB + 1) * (sizeof(LsePartial) + sizeof(double2)) + smc_lse_scratch_bytes() + 1024;
}

// workspace: [LsePartial nb+1][double2 nb+1][finalize scratch]
static void *pf_scratch(void *ws, int nb)
{
    size_t o = ((size_t)(nb + 1) * sizeof(LsePartial) + 255) & ~(size_t)255;
    o += ((size_t)(nb + 1) * sizeof(double2) + 255) & ~(size_t)255;
    return (char *)ws + o;
}

static int pf_check(double *x, double *lw_raw, int64_t n, uint64_t *ctrs, const double *obs, smc_wstate *st,
                    void *ws, size_t ws_bytes, const char *who)
{
    if (!x || !lw_raw || !ctrs || !obs || !st || n < 1 || n >= ((int64_t)1 << 31))
        return smc_set_error(SMC_EINVAL, "%s: bad args", who);
    if ((uintptr_t)x & 31) return smc_set_error(SMC_EINVAL, "%s: state must be 32-byte aligned", who);
    if (!ws || ws_bytes < smc_pf_workspace_bytes(n)) return smc_set_error(SMC_EWORKSPACE, "%s: workspace", who);
    return SMC_OK;
}

extern "C" int smc_pf_init(double *x, double *lw_raw, int64_t n, uint64_t stream_base, uint64_t seed, uint64_t *ctrs,
                           const double *obs_t, smc_wstate *st, double *partial_out, void *ws, size_t ws_bytes,
                           void *stream)
{
    int rc = pf_check(x, lw_raw, n, ctrs, obs_t, st, ws, ws_bytes, "smc_pf_init");
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = (int)((n + PB - 1) / PB);
    LsePartial *parts = (LsePartial *)ws;
    void *scratch = pf_scratch(ws, nb);
    smc_launch(k_pf_init, nb, PB, 0, s, x, lw_raw, n, stream_base, make_key_sched(seed), ctrs, obs_t,
                                pf_constants(), st, parts);
    smc_launch_lse_finalize(parts, nb, st, n, SMC_W_SET_LOG, 1, s, scratch, nullptr, nullptr, partial_out);
    return smc_check_launch("smc_pf_init");
}

static int pf_move(const double *x_in, double *x, const int32_t *parents, const int32_t *gate, double *lw_raw,
                   int64_t n, uint64_t stream_base, int64_t n_total, uint64_t seed, uint64_t *ctrs, const uint64_t *ctr_u,
                   const double *obs_t, smc_wstate *st, double *incw_out, double *monitor_prev, double *partial_out,
                   void *ws, size_t ws_bytes, void *stream, const char *who)
{
    uint64_t dummy = 0;
    int rc = pf_check(x, lw_raw, n, ctr_u ? &dummy : ctrs, obs_t, st, ws, ws_bytes, who);
    if (rc) return rc;
    if (ctr_u && (uint32_t)*ctr_u > 0xFFFFFFFFu - 15u)
        return smc_set_error(SMC_EINVAL, "%s: uniform counter would carry into its high word", who);
    if (ctr_u && stream_base + (uint64_t)n > ((uint64_t)1 << 32))
        return smc_set_error(SMC_EINVAL, "%s: uniform counts need stream indices below 2^32", who);
    if (!x_in) x_in = x;
    if ((uintptr_t)x_in & 31) return smc_set_error(SMC_EINVAL, "%s: x_in must be 32-byte aligned", who);
    if (parents && x_in == x)
        return smc_set_error(SMC_EINVAL, "%s: a gathering move needs distinct in/out state buffers", who);
    cudaStream_t s = (cudaStream_t)stream;
    // PF_PPT particles per thread only while the grid still gives every SM >= 4 blocks;
    // below that (e.g. config 1, N = 10^4) one particle per thread spreads the latency
    const bool many = n >= (int64_t)MB * 148 * 4;
    const int nb = (int)(many ? (n + MB - 1) / MB : (n + PB - 1) / PB);
    LsePartial *parts = (LsePartial *)ws;
    double2 *mon = (double2 *)((char *)ws + (((size_t)(nb + 1) * sizeof(LsePartial) + 255) & ~(size_t)255));
    void *scratch = pf_scratch(ws, nb);
    const KeySched key = make_key_sched(seed);
    const double w_eq = 1.0 / (double)(n_total > 0 ? n_total : n);
    const UniformCtr cu = make_uniform_ctr(ctr_u ? *ctr_u : 0, key);
#define SMC_PF_MOVE(MONV, PPTV, MONP)                                                                          \
    do {                                                                                                       \
        if (h_move_ws && PPTV == PF_PPT && PB == WSC) {                                                        \
            if (ctr_u)                                                                                         \
                smc_launch(k_pf_move_ws<MONV, PF_PPT, true>, nb, WST, 0, s, x_in, x, parents, gate, lw_raw, n,  \
                           stream_base, w_eq, key, ctrs, cu, obs_t, pf_constants(), st, incw_out, parts, MONP); \
            else                                                                                               \
                smc_launch(k_pf_move_ws<MONV, PF_PPT, false>, nb, WST, 0, s, x_in, x, parents, gate, lw_raw, n, \
                           stream_base, w_eq, key, ctrs, cu, obs_t, pf_constants(), st, incw_out, parts, MONP); \
        } else if (ctr_u)                                                                                      \
            smc_launch(k_pf_move<MONV, PPTV, true>, nb, PB, 0, s, x_in, x, parents, gate, lw_raw, n, stream_base, \
                       w_eq, key, ctrs, cu, obs_t, pf_constants(), st, incw_out, parts, MONP);                \
        else                                                                                                   \
            smc_launch(k_pf_move<MONV, PPTV, false>, nb, PB, 0, s, x_in, x, parents, gate, lw_raw, n, stream_base, \
                       w_eq, key, ctrs, cu, obs_t, pf_constants(), st, incw_out, parts, MONP);                \
    } while (0)
    if (monitor_prev) {
        if (many) SMC_PF_MOVE(true, PF_PPT, mon); else SMC_PF_MOVE(true, 1, mon);
        smc_launch_lse_finalize(parts, nb, st, n, SMC_W_ADD_LOG, 1, s, scratch, mon, monitor_prev, partial_out);
    } else {
        if (many) SMC_PF_MOVE(false, PF_PPT, nullptr); else SMC_PF_MOVE(false, 1, nullptr);
        smc_launch_lse_finalize(parts, nb, st, n, SMC_W_ADD_LOG, 1, s, scratch, nullptr, nullptr, partial_out);
    }
#undef SMC_PF_MOVE
    return smc_check_launch(who);
}

extern "C" int smc_pf_move(const double *x_in, double *x, const int32_t *parents, const int32_t *gate, double *lw_raw,
                           int64_t n, uint64_t stream_base, int64_t n_total, uint64_t seed, uint64_t *ctrs,
                           const double *obs_t, smc_wstate *st, double *incw_out, double *monitor_prev,
                           double *partial_out, void *ws, size_t ws_bytes, void *stream)
{
    return pf_move(x_in, x, parents, gate, lw_raw, n, stream_base, n_total, seed, ctrs, nullptr, obs_t, st, incw_out,
                   monitor_prev, partial_out, ws, ws_bytes, stream, "smc_pf_move");
}

extern "C" int smc_pf_move_uniform(const double *x_in, double *x, const int32_t *parents, const int32_t *gate,
                                   double *lw_raw, int64_t n, uint64_t stream_base, int64_t n_total, uint64_t seed,
                                   uint64_t ctr, const double *obs_t, smc_wstate *st, double *incw_out,
                                   double *monitor_prev, double *partial_out, void *ws, size_t ws_bytes, void *stream)
{
    return pf_move(x_in, x, parents, gate, lw_raw, n, stream_base, n_total, seed, nullptr, &ctr, obs_t, st, incw_out,
                   monitor_prev, partial_out, ws, ws_bytes, stream, "smc_pf_move_uniform");
}

int smc_pf_set_move_ws(int on)  // smc_debug_set(SMC_DEBUG_MOVE_WS, on) (A/B and the bit-identity test)
{
    h_move_ws = on;
    return SMC_OK;
}
