// smc_resample.cu -- resampling on sm_100a (replaces smckit.resample, SPEC.md:114-199,
// and the value collection's copy, SPEC.md:342-349 / PAPER.md:418-433).
//
// Pinned integer contract, shared bit-for-bit
// with oracle/smc_oracle.c:
//   q_i = floor(W_i 2^63), Q = inclusive prefix, T = Q_{N-1}, |T - 2^63| <= 2^43
//   stratified/systematic over M strata: P_k = floor((k + m_k 2^-53) T / M)
//   multinomial:                          P_k = floor(m_k T 2^-53)
//   particle i receives #{k : Q_{i-1} <= P_k < Q_i}   (strict bound)
//   residual: f_i = floor(fl(M W_i)); the R = M - sum f leftovers over
//   q'_i = floor((fl(M W_i) - f_i) 2^(63 - ceil log2 N)).
//
// Kernels (one stratified/systematic resample = 4 launches):
//   A  k_rs_tiles   : per-tile u128 sums of q, sums of f and q'; validation.
//   S  k_rs_scan    : one block: T, R, window check, tile prefixes, the stream
//                     counter advance (on device: no host sync).
//  [M  k_rs_prefix + k_mn_{count,scan,scatter,assign}: multinomial/residual histogram
//      with the draws bucketed by tile]
//   B  k_rs_counts  : per tile (coalesced loads staged through shared memory),
//                     local scan + tile prefix -> Q; counts in O(1) per particle
//                     via F(X) = #{k : P_k < X} (fp64 with a guard band, exact
//                     128-bit fallback inside it) and the tile's (zero slots,
//                     surplus parents, surplus children) aggregate.
//   S2 k_rs_zsp_scan: one block: exclusive prefixes of those aggregates.
//   B2 k_rs_ranks   : per tile: the compacted surplus-parent list + rank anchors.
//   C  k_rs_assign  : per slot tile: the slice of the surplus-parent list that
//                     covers the tile's zero ranks (located through the rank
//                     anchors) staged in shared memory, each staged parent writes
//                     itself into the tile's rank table, every zero slot reads its
//                     parent by rank; with 32-byte rows the in-place row copy is
//                     fused in (256-bit LDG/STG, 4 rows in flight per thread).
#include "smc_weights.cuh"

using namespace smc;

namespace {

constexpr int RT = 256;
#ifndef RS_TILES_MINB_W
#define RS_TILES_MINB_W 8  // pass A from an explicit W vector, not residual: 8 blocks/SM (32 registers)
#endif
#ifndef RS_TILES_MINB
#define RS_TILES_MINB 6  // pass A: 6 blocks/SM (40 registers, no spills of the branch-free item loop)
#endif
#ifndef RS_COUNTS_MINB
#define RS_COUNTS_MINB 5  // pass B1 blocks per SM the register allocation must allow (same-box A/B: 5 > 6 > 4)
#endif
constexpr int RI = 8;
constexpr int TILE = RT * RI;  // elements per tile (pass A/B) and ranks per tile (pass C)
constexpr uint64_t T_LO = (1ull << 63) - (1ull << 43);
constexpr uint64_t T_HI = (1ull << 63) + (1ull << 43);
constexpr double TWO53 = 9007199254740992.0;
constexpr double INV53 = 1.0 / 9007199254740992.0;
constexpr int ANCHOR = 64;  // rank granularity of the surplus-parent anchors (pass B2 -> C)

__device__ int g_force_exact = 0;  // test hook: always take the exact 128-bit F path

struct RsHeader {
    uint64_t T;       // sum of q
    uint64_t Tm;      // total of the CDF that is searched (T or T')
    uint64_t M;       // positions (strata / draws)
    uint64_t c0;      // first counter of the resampling stream for this call
    uint64_t m_sys;   // the single systematic uniform (53-bit integer)
    double ratio;     // fl(M / Tm) for the fast F path
    double guard;     // guard band of the fast F path
    int64_t draws;
    int32_t active;   // 0 => gated off or failed; later kernels exit
    int32_t trivial;  // N == 1
    uint32_t Z_total, S_total, P_total;
    uint64_t qoff;    // this shard's CDF offset (0 on one GPU)
    int32_t mn_direct;  // multinomial: a position bin overflowed its capacity -> direct search
    double mn_rb;       // multinomial: 2^kb / Tm (bin-boundary estimate, exact fix-up)
};

struct MnGeom {
    int kb;
    int64_t nb, cap;
};

struct Layout {
    RsHeader *hdr;
    SMC_DEV RsHeader *hdr_w() const { return hdr; }
    u128 *tile_q;
    int64_t *tile_f;
    uint64_t *tile_qr;
    uint64_t *tile_pre;
    uint64_t *tile_zsp;  // per slot tile: packed (zero slots, surplus parents, surplus children)
    uint4 *tile_excl;   // per slot tile: exclusive (Z, S, P) prefix
    int32_t *anchor, *sp_idx, *sp_start;  // anchor[k]: surplus parent covering rank k*ANCHOR
    int32_t *tile_z0;   // per slot tile: its first zero rank (and Z at index nt)
    uint32_t *zmask;    // zero-count slots, one bit per slot (TILE / 32 words per tile), for pass C
    uint64_t *qfull;
    int32_t *cnt;       // multinomial histogram, then the counts when the caller passes none
    uint32_t *mn_fill;  // multinomial: positions per bin (reserved runs)
    uint64_t *mn_pos;   // multinomial: positions by bin, `cap` slots per bin
    uint32_t *mn_start; // multinomial: first particle reached by every bin's positions (B + 1)
    uint32_t *mn_cnt, *mn_off;  // MN1: draws per position bin, bin offsets in mn_pos
    MnGeom mg;                  // MN2 bin geometry of this n (mn_geom, evaluated on the host)
    size_t bytes;
};

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// Multinomial position bins: B = 2^kb bins by the top kb bits of the 53-bit draw m (the
// position P = floor(m Tm / 2^53) is monotone in m, so bin b holds exactly the positions
// [floor(b Tm / 2^kb), ~floor((b+1) Tm / 2^kb)] -- no division, no search), ~8192
// positions per bin (at most 4096 bins), and a fixed capacity of cap slots per bin (the
// draws' bins are Binomial(M, 2^-kb) whatever the weights: mean + 8 sd + 64; an overflow --
// adversarial explicit uniforms -- falls back to the direct search).
__host__ __device__ inline MnGeom mn_geom(int64_t n)
{
    MnGeom g;
    g.kb = 0;
    while (g.kb < 12 && (n >> g.kb) > 8192) ++g.kb;
    g.nb = (int64_t)1 << g.kb;
    const int64_t per = (n + g.nb - 1) / g.nb;
    int64_t sd = (int64_t)sqrt((double)per);  // ceil(sqrt(per)): correctly rounded sqrt, one fix-up
    while (sd * sd < per) ++sd;
    g.cap = per + 8 * sd + 64;
    return g;
}

// The binned kernels' shared memory (k_mn2_scatter: a block's 12288 draws (10 B each) + 3 words per bin;
// k_mn2_count: a bin's `cap` positions + 2 x 8193 sub-bucket words).  Past N ~ 2^26 a bin no
// longer fits one block's shared memory: those N take the global-memory bucket path (MN1).
constexpr int MT = 1024;          // threads of the multinomial kernels
// draws per thread in k_mn2_scatter: 6 while the block's shared memory (10 B per draw + 12 B per
// bin) lets two blocks share an SM (<= 2048 bins, N <= 2^24), else 12 (same-box A/B,
// profiles/r2_resample_ab.txt)
__host__ __device__ inline int mn_dpt(int64_t nb) { return nb <= 2048 ? 6 : 12; }
constexpr int NSB = 4096;         // most sub-buckets of a bin in k_mn2_count (~2 positions each)
#ifndef MN_SCATTER_MINB
#define MN_SCATTER_MINB 2  // k_mn2_scatter<6> blocks per SM (2: 32 registers, the draws' positions partly spilled)
#endif
#ifndef MN_FU
#define MN_FU 4  // positions of a sub-bucket k_mn2_count's F(X) checks predicated before its remainder loop
#endif
constexpr size_t MN_SMEM_MAX = 232448;  // 227 KB: the sm_100 per-block opt-in maximum
__host__ __device__ inline size_t mn2_scatter_smem(int64_t n)
{
    const MnGeom g = mn_geom(n);
    return (size_t)MT * mn_dpt(g.nb) * (8 + 2) + (size_t)g.nb * 12 + 64;
}
__host__ __device__ inline size_t mn2_count_smem(int64_t n)
{
    return (size_t)mn_geom(n).cap * 8 + (size_t)(NSB + 1) * 4 * 2 + 64;
}
__host__ __device__ inline bool mn2_fits(int64_t n)
{
    return mn2_scatter_smem(n) <= MN_SMEM_MAX && mn2_count_smem(n) <= MN_SMEM_MAX;
}
// MN1 (N past mn2_fits): ~256 particles per position bin, at most 2^17 bins
constexpr int64_t MN1_MAX_BINS = 1 << 17;
__host__ __device__ inline int64_t mn1_bins(int64_t n)
{
    const int64_t b = (n + 255) / 256;
    return b < MN1_MAX_BINS ? b : MN1_MAX_BINS;
}

Layout layout(void *ws, int64_t n)
{
    const int64_t nt = (n + TILE - 1) / TILE;
    char *p = (char *)ws;
    Layout L;
    size_t o = 0;
    auto take = [&](size_t b) { char *r = p ? p + o : nullptr; o += al(b); return (void *)r; };
    L.hdr = (RsHeader *)take(sizeof(RsHeader));
    L.tile_q = (u128 *)take(sizeof(u128) * nt);
    L.tile_f = (int64_t *)take(sizeof(int64_t) * nt);
    L.tile_qr = (uint64_t *)take(sizeof(uint64_t) * nt);
    L.tile_pre = (uint64_t *)take(sizeof(uint64_t) * nt);
    L.tile_zsp = (uint64_t *)take(sizeof(uint64_t) * nt);
    L.tile_excl = (uint4 *)take(sizeof(uint4) * (nt + 1));
    L.anchor = (int32_t *)take(sizeof(int32_t) * (n / ANCHOR + 2));
    L.sp_idx = (int32_t *)take(sizeof(int32_t) * (n + 1));  // P <= n even for invalid counts
    L.sp_start = (int32_t *)take(sizeof(int32_t) * (n + 2));
    L.tile_z0 = (int32_t *)take(sizeof(int32_t) * (nt + 2));
    L.zmask = (uint32_t *)take(sizeof(uint32_t) * nt * (TILE / 32));
    L.qfull = (uint64_t *)take(sizeof(uint64_t) * n);
    L.cnt = (int32_t *)take(sizeof(int32_t) * n);
    const MnGeom mg = mn_geom(n);
    L.mg = mg;
    const bool mn2 = mn2_fits(n);
    const int64_t nb1 = mn2 ? 0 : mn1_bins(n), nbm = mg.nb > nb1 ? mg.nb : nb1;
    L.mn_fill = (uint32_t *)take(sizeof(uint32_t) * (nbm + 1));
    L.mn_pos = (uint64_t *)take(sizeof(uint64_t) * (mn2 ? mg.nb * mg.cap : n));  // MN1: capacity n positions
    L.mn_start = (uint32_t *)take(sizeof(uint32_t) * (nbm + 2));
    L.mn_cnt = (uint32_t *)take(sizeof(uint32_t) * (nb1 + 1));
    L.mn_off = (uint32_t *)take(sizeof(uint32_t) * (nb1 + 1));
    L.bytes = o;
    return L;
}

// Everything a per-particle kernel needs to turn an index into W_i.
struct WSrc {
    const double *w;   // normalized weights, or null
    const double *lw;  // raw log weights (w == null)
    const smc_wstate *st;
    int64_t n;
    SMC_DEV NormLw norm() const { return w ? NormLw{0.0, 0.0, false, 0.0} : norm_of(st); }
    SMC_DEV double raw(int64_t i, const NormLw &nl) const  // the load (coalescable)
    {
        if (w) return __ldg(w + i);
        return nl.eq ? 0.0 : __ldg(lw + i);
    }
    SMC_DEV double weight(double r, const NormLw &nl, const smc_fm::ExpEntry *tab = smc_fm::kExpTab) const
    {
        if (w) return r;
        return weight_of_lw(r, nl, tab);
    }
    // W = exp(lw - lse): the table exp (<= 0.52 ulp, 6 fp64 operations fewer than a
    // table-free polynomial; below 2^-1022 it flushes to +0, which is what floor(W 2^63)
    // makes of it anyway).  smc_weights_read uses this same function, so the weights a
    // caller reads are bit for bit the ones the resampler quantizes.
    SMC_DEV static double weight_of_lw(double r, const NormLw &nl, const smc_fm::ExpEntry *tab)
    {
        return nl.eq ? nl.weq : smc_fm::exp_nonpos_cb(nl(r), tab);
    }
};

// The exp table (2 KB) staged in shared memory by a block: requested before the
// dependency wait (constant data), stored, and published by the block's next barrier.
struct ExpTabStage {
    double2 v;
    SMC_DEV void load()
    {
        if (threadIdx.x < 128) v = __ldg(reinterpret_cast<const double2 *>(smc_fm::kExpTab) + threadIdx.x);
    }
    SMC_DEV void store(smc_fm::ExpEntry *t) const
    {
        if (threadIdx.x < 128) reinterpret_cast<double2 *>(t)[threadIdx.x] = v;
    }
};

SMC_DEV bool is_residual(int scheme)
{
    return scheme == SMC_RESIDUAL || scheme == SMC_RESIDUAL_STRATIFIED || scheme == SMC_RESIDUAL_SYSTEMATIC;
}
SMC_DEV bool is_multinomial(int scheme) { return scheme == SMC_MULTINOMIAL || scheme == SMC_RESIDUAL; }
SMC_DEV bool is_systematic(int scheme) { return scheme == SMC_SYSTEMATIC || scheme == SMC_RESIDUAL_SYSTEMATIC; }

// q, f, q' for one weight (A.1, A.4).  Validation sets `bad`.
struct Quant {
    uint64_t q, qr;
    int64_t f;
};
SMC_DEV Quant quantize(double W, bool residual, double m_out, double rscale, bool &bad)
{
    Quant r{0, 0, 0};
    const uint64_t wb = smc_fm::bits(W);  // W in [0, 1]: bits <= bits(1.0) (or -0); NaN / < 0 / > 1 are not
    if (wb > 0x3FF0000000000000ull && wb != 0x8000000000000000ull) { bad = true; return r; }
    r.q = (uint64_t)(W * 9223372036854775808.0);
    if (residual) {
        const double x = m_out * W;  // fl(M W_i), exactly rounded (no FMA: --fmad=false)
        const double f = floor(x);
        r.f = (int64_t)f;
        r.qr = (uint64_t)((x - f) * rscale);
    }
    return r;
}

// ------------------------------------------------------------------ pass A --
// LW: the weights come from the raw log weights + the weight record (the sampler's
// path: the table exp staged in shared memory); otherwise from an explicit W vector.
template <bool RES, bool MULTI, bool LW>  // scheme family and weight source: resolved at compile time
__global__ void __launch_bounds__(RT, LW || RES ? RS_TILES_MINB : RS_TILES_MINB_W) k_rs_tiles(int scheme, WSrc src, int64_t n, double m_out, double rscale,
                                                 const double *__restrict__ u, int64_t n_u, const int32_t *gate,
                                                 int32_t *status, Layout L)
{
    __shared__ smc_fm::ExpEntry s_tab[128];
    ExpTabStage ts;
    if (LW) ts.load();
    SMC_PDL_WAIT();
    if (gate && *gate == 0) return;
    const int64_t base = (int64_t)blockIdx.x * TILE;
    const NormLw nl = src.norm();
    const bool full = base + TILE <= n;  // no per-element bounds checks on full tiles
    const int rem = full ? TILE : (int)(n - base);
    // 32-bit offsets from the tile's base pointers (no 64-bit index arithmetic per element)
    const double *g = LW ? (nl.eq ? nullptr : src.lw + base) : src.w + base;
    uint64_t *qb = L.qfull + base;
    double r[RI];
#pragma unroll
    for (int j = 0; j < RI; ++j) {  // striped: each warp load is 256 contiguous bytes; all issued up front
        const int li = j * RT + threadIdx.x;
        r[j] = (g && (full || li < rem)) ? __ldg(g + li) : 0.0;
    }
    if (LW) {
        ts.store(s_tab);
        __syncthreads();
    }
    u128 sq = 0;
    uint64_t sqr = 0;
    int64_t sf = 0;
    bool anybad = false;
    // branch-free over the RI items (items past the end: W = 0, q = 0; stores predicated); a bad
    // weight (NaN, < 0, > 1) fails the call, so what it adds to the sums does not matter
#pragma unroll
    for (int j = 0; j < RI; ++j) {
        const int li = j * RT + threadIdx.x;
        const bool in = full || li < rem;
        double W = LW ? WSrc::weight_of_lw(r[j], nl, s_tab) : r[j];
        W = in ? W : 0.0;
        const uint64_t wb = smc_fm::bits(W);
        anybad |= wb > 0x3FF0000000000000ull && wb != 0x8000000000000000ull;
        const uint64_t q = (uint64_t)(W * 9223372036854775808.0);  // floor(W 2^63), A.1
        uint64_t qr = 0;
        int32_t fi = 0;
        sq += q;
        if (RES) {
            const double x = m_out * W;  // fl(M W_i), exactly rounded (no FMA: --fmad=false)
            const double f = floor(x);
            qr = (uint64_t)((x - f) * rscale);
            sqr += qr;
            sf += (int64_t)f;
            fi = (int32_t)f;
        }
        if (in) {
            qb[li] = RES ? qr : q;  // the searched quantity, for passes M and B1
            // the draws' histogram starts from the residual floors f_i (0 for multinomial): the
            // draw kernels add onto it, and pass B1 reads the finished counts without re-deriving f
            if (MULTI || RES) L.cnt[base + li] = fi;  // residual-stratified / -systematic: B1 reads f_i here
        }
    }
    if (__any_sync(0xffffffffu, anybad)) {  // rare: name the first bad weight
#pragma unroll
        for (int j = 0; j < RI; ++j) {
            const int li = j * RT + threadIdx.x;
            if (!(full || li < rem)) continue;
            const double rr = g ? __ldg(g + li) : 0.0;  // reloaded: the item registers are not kept live
            bool bad = false;
            quantize(LW ? WSrc::weight_of_lw(rr, nl, s_tab) : rr, RES, m_out, rscale, bad);
            if (bad) raise_status_at(status, SMC_EUNNORMALIZED, base + li);
        }
    }
    // explicit uniforms must lie in [0, 1) (the index reported is the uniform's)
    for (int64_t k = (int64_t)blockIdx.x * RT + threadIdx.x; u && k < n_u; k += (int64_t)gridDim.x * RT)
        if (!(u[k] >= 0.0 && u[k] < 1.0)) raise_status_at(status, SMC_EINVAL, k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += shfl_xor_u128(sq, o);
        if (RES) {
            sqr += __shfl_xor_sync(0xffffffffu, sqr, o);
            sf += __shfl_xor_sync(0xffffffffu, sf, o);
        }
    }
    __shared__ u128 s_q[RT / 32];
    __shared__ uint64_t s_qr[RT / 32];
    __shared__ int64_t s_f[RT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_q[warp] = sq; s_qr[warp] = sqr; s_f[warp] = sf; }
    __syncthreads();
    if (threadIdx.x == 0) {
        u128 a = 0;
        uint64_t b = 0;
        int64_t c = 0;
        for (int w = 0; w < RT / 32; ++w) { a += s_q[w]; b += s_qr[w]; c += s_f[w]; }
        L.tile_q[blockIdx.x] = a;
        L.tile_qr[blockIdx.x] = b;
        L.tile_f[blockIdx.x] = c;
    }
}

inline void launch_tiles(int scheme, unsigned nt, cudaStream_t s, WSrc src, int64_t n, double mo, double rscale,
                         const double *u, int64_t n_u, const int32_t *gate, int32_t *status, Layout L)
{
    const bool res = scheme == SMC_RESIDUAL || scheme == SMC_RESIDUAL_STRATIFIED || scheme == SMC_RESIDUAL_SYSTEMATIC;
    const bool multi = scheme == SMC_MULTINOMIAL || scheme == SMC_RESIDUAL;
#define SMC_TILES(R_, M_)                                                                                              \
    (src.w ? smc_launch(k_rs_tiles<R_, M_, false>, nt, RT, 0, s, scheme, src, n, mo, rscale, u, n_u, gate, status, L) \
           : smc_launch(k_rs_tiles<R_, M_, true>, nt, RT, 0, s, scheme, src, n, mo, rscale, u, n_u, gate, status, L))
    if (res && multi) SMC_TILES(true, true);
    else if (res) SMC_TILES(true, false);
    else if (multi) SMC_TILES(false, true);
    else SMC_TILES(false, false);
#undef SMC_TILES
}

// ------------------------------------------------------------------ pass S --
constexpr int SB = 1024;

// A shard's totals {T lo, T hi, sum f, T'} for the allgather of a G-GPU resample.
__global__ void __launch_bounds__(SB) k_rs_local_totals(int64_t nt, const int32_t *gate, Layout L, uint64_t *out)
{
    SMC_PDL_WAIT();
    __shared__ u128 s_q[SB / 32];
    __shared__ uint64_t s_qr[SB / 32];
    __shared__ int64_t s_f[SB / 32];
    if (gate && *gate == 0) {
        if (threadIdx.x == 0) { out[0] = out[1] = out[2] = out[3] = 0; }
        return;
    }
    u128 tq = 0;
    uint64_t tqr = 0;
    int64_t tf = 0;
    for (int64_t b = threadIdx.x; b < nt; b += SB) { tq += L.tile_q[b]; tqr += L.tile_qr[b]; tf += L.tile_f[b]; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tq += shfl_xor_u128(tq, o);
        tqr += __shfl_xor_sync(0xffffffffu, tqr, o);
        tf += __shfl_xor_sync(0xffffffffu, tf, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_q[warp] = tq; s_qr[warp] = tqr; s_f[warp] = tf; }
    __syncthreads();
    if (threadIdx.x == 0) {
        u128 T = 0;
        uint64_t Tr = 0;
        int64_t F = 0;
        for (int w = 0; w < SB / 32; ++w) { T += s_q[w]; Tr += s_qr[w]; F += s_f[w]; }
        out[0] = (uint64_t)T;
        out[1] = (uint64_t)(T >> 64);
        out[2] = (uint64_t)F;
        out[3] = Tr;
    }
}

// totals_all != NULL: a shard of a G-GPU system -- the global T / sum f / T'
// come from the allgathered per-shard totals (4 u64 each: T lo, T hi, sum f, T'),
// and this shard's CDF starts at the exact integer offset of the shards before it.
__global__ void __launch_bounds__(SB) k_rs_scan(int scheme, int64_t n, int64_t nt, uint64_t m_out, Key key,
                                                uint64_t stream, uint64_t *ctr, const double *__restrict__ u,
                                                int64_t n_u, const int32_t *gate, int32_t *status, Layout L,
                                                const uint64_t *totals_all, int G, int rank, int64_t n_total)
{
    SMC_PDL_WAIT();
    __shared__ uint64_t s_off;
    __shared__ uint64_t sm64[SB / 32 + 1];
    __shared__ u128 s_q[SB / 32];
    __shared__ uint64_t s_qr[SB / 32];
    __shared__ int64_t s_f[SB / 32];
    __shared__ int s_ok;
    RsHeader *h = L.hdr;
    if (gate && *gate == 0) {
        if (threadIdx.x == 0) h->active = 0;
        return;
    }
    const bool residual = is_residual(scheme);
    // totals: striped, so every warp load is coalesced (integer sums are order independent);
    // 8 tiles per thread per round, all loads issued before any is consumed (one round trip
    // per round instead of one per tile)
    constexpr int KS = 8;
    u128 tq = 0;
    uint64_t tqr = 0;
    int64_t tf = 0;
    for (int64_t b0 = threadIdx.x; b0 < nt; b0 += (int64_t)KS * SB) {
        u128 vq[KS];
        uint64_t vr[KS];
        int64_t vf[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            const int64_t b = b0 + (int64_t)k * SB;
            vq[k] = b < nt ? L.tile_q[b] : (u128)0;
            vr[k] = residual && b < nt ? L.tile_qr[b] : 0;
            vf[k] = residual && b < nt ? L.tile_f[b] : 0;
        }
#pragma unroll
        for (int k = 0; k < KS; ++k) { tq += vq[k]; tqr += vr[k]; tf += vf[k]; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tq += shfl_xor_u128(tq, o);
        tqr += __shfl_xor_sync(0xffffffffu, tqr, o);
        tf += __shfl_xor_sync(0xffffffffu, tf, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_q[warp] = tq; s_qr[warp] = tqr; s_f[warp] = tf; }
    __syncthreads();
    if (threadIdx.x == 0) {
        u128 T = 0;
        uint64_t Tr = 0;
        int64_t F = 0;
        for (int w = 0; w < SB / 32; ++w) { T += s_q[w]; Tr += s_qr[w]; F += s_f[w]; }
        uint64_t off = 0;
        if (totals_all) {
            T = 0; Tr = 0; F = 0;
            for (int g = 0; g < G; ++g) {
                const uint64_t *t4 = totals_all + 4 * g;
                const u128 Tg = ((u128)t4[1] << 64) | t4[0];
                if (g < rank) off += residual ? t4[3] : t4[0];
                T += Tg;
                F += (int64_t)t4[2];
                Tr += t4[3];
            }
        }
        s_off = off;
        h->qoff = off;
        int ok = (status == nullptr || *status == 0);
        if (T < (u128)T_LO || T > (u128)T_HI) { raise_status(status, SMC_EUNNORMALIZED); ok = 0; }
        int64_t M = (int64_t)m_out;
        uint64_t Tm = (uint64_t)T;
        if (ok && residual && n_total > 1) {
            M = (int64_t)m_out - F;
            if (M < 0) { raise_status(status, SMC_EUNNORMALIZED); ok = 0; }
            if (M > 0 && Tr == 0) { raise_status(status, SMC_EUNNORMALIZED); ok = 0; }
            Tm = Tr;
        }
        int64_t draws = 0;
        if (n_total > 1 && M > 0) draws = is_systematic(scheme) ? 1 : M;
        if (ok && u && n_u < draws) { raise_status(status, SMC_EUNIFORMS); ok = 0; }
        h->T = (uint64_t)T;
        h->Tm = Tm;
        h->M = (uint64_t)(M > 0 ? M : 0);
        h->ratio = Tm ? (double)(M > 0 ? M : 0) / (double)Tm : 0.0;
        // |fl(X) fl(M/Tm) - X M/Tm| <= 3.4e-16 * M; flag anything within 2^-47 M of a decision boundary
        h->guard = (double)(M > 0 ? M : 1) * 7.105427357601002e-15;
        h->draws = draws;
        h->trivial = (n_total == 1);
        h->Z_total = h->S_total = h->P_total = 0;
        if (ok) {
            const uint64_t c0 = u ? 0 : *ctr;
            h->c0 = c0;
            if (!u) *ctr = c0 + (uint64_t)draws;
            if (is_systematic(scheme))
                h->m_sys = draws ? (u ? (uint64_t)(u[0] * TWO53) : draw53(c0, stream, key)) : 0;
        }
        h->active = ok;
        h->mn_direct = 0;
        h->mn_rb = Tm ? ldexp(1.0, L.mg.kb) / (double)Tm : 0.0;
        s_ok = ok;
    }
    if (is_multinomial(scheme)) {  // the multinomial bins: empty, every start at the last particle
        const MnGeom g = L.mg;  // host-computed (Layout)
        for (int64_t b = threadIdx.x; b <= g.nb; b += SB) {
            L.mn_fill[b] = 0;
            L.mn_start[b] = (uint32_t)(n - 1);
        }
    }
    __syncthreads();
    if (!s_ok) return;
    // exclusive prefix of the searched per-tile totals (all < 2^64 once T is validated):
    // warp w owns a contiguous chunk; its lanes read consecutive tiles (coalesced) and
    // scan them 32 at a time with a running carry, offset by the warps before it.
    constexpr int NW = SB / 32;
    const int64_t C = (nt + NW - 1) / NW;
    const int64_t w0 = warp * C < nt ? warp * C : nt, w1 = w0 + C < nt ? w0 + C : nt;
    auto val = [&](int64_t b) { return residual ? L.tile_qr[b] : (uint64_t)L.tile_q[b]; };
    uint64_t wsum = 0;
    for (int64_t b0 = w0 + lane; b0 < w1; b0 += 32 * KS) {
        uint64_t v[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) v[k] = b0 + 32 * k < w1 ? val(b0 + 32 * k) : 0;
#pragma unroll
        for (int k = 0; k < KS; ++k) wsum += v[k];
    }
    wsum = warp_sum(wsum);
    if (lane == 0) sm64[warp] = wsum;
    __syncthreads();
    if (warp == 0) {
        const uint64_t x = sm64[lane];
        const uint64_t inc = warp_inclusive_sum(x);
        sm64[lane] = inc - x;
    }
    __syncthreads();
    uint64_t carry = sm64[warp] + s_off;
    for (int64_t c0 = w0; c0 < w1; c0 += 32 * KS) {  // KS warp-rows in flight, then scanned in order
        uint64_t v[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            const int64_t b = c0 + 32 * k + lane;
            v[k] = b < w1 ? val(b) : 0;
        }
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            const int64_t b = c0 + 32 * k + lane;
            const uint64_t inc = warp_inclusive_sum(v[k]);
            if (b < w1) L.tile_pre[b] = carry + inc - v[k];
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
}

// One GPU, nt <= 8 SB tiles (N <= 2^24): the same results as k_rs_scan in ONE pass over the
// tile sums -- each lane keeps its <= 8 tiles (the chunked layout the scan needs) in registers
// for both the totals and the scan, the block reduction ends in warp shuffles instead of a
// serial loop, and the header's dependent loads (status, stream counter) are issued at entry.
template <bool RES>
__global__ void __launch_bounds__(SB) k_rs_scan1(int scheme, int64_t n, int64_t nt, uint64_t m_out, Key key,
                                                 uint64_t stream, uint64_t *ctr, const double *__restrict__ u,
                                                 int64_t n_u, const int32_t *gate, int32_t *status, Layout L)
{
    SMC_PDL_WAIT();
    RsHeader *h = L.hdr;
    if (gate && *gate == 0) {
        if (threadIdx.x == 0) h->active = 0;
        return;
    }
    __shared__ u128 s_q[SB / 32];
    __shared__ uint64_t s_qr[SB / 32], s_w[SB / 32];
    __shared__ int64_t s_f[SB / 32];
    __shared__ int s_ok;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t st0 = 0;
    uint64_t c00 = 0;
    if (threadIdx.x == 0) {  // the header's own loads, in flight while the tiles are summed
        st0 = status ? *status : 0;
        c00 = u ? 0 : *ctr;
    }
    constexpr int NW = SB / 32, KS = 8;
    const int64_t C = (nt + NW - 1) / NW;  // <= 8 * 32: warp w owns tiles [w C, (w+1) C)
    const int64_t w0 = min((int64_t)warp * C, nt), w1 = min(w0 + C, nt);
    uint64_t v[KS];
    u128 tq = 0;
    uint64_t tqr = 0, wsum = 0;
    int64_t tf = 0;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
        const int64_t b = w0 + 32 * k + lane;
        const bool in = b < w1;
        const u128 q = in ? L.tile_q[b] : (u128)0;
        const uint64_t qr = RES && in ? L.tile_qr[b] : 0;
        tq += q;
        if (RES) {
            tqr += qr;
            tf += in ? L.tile_f[b] : 0;
        }
        v[k] = RES ? qr : (uint64_t)q;
        wsum += v[k];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tq += shfl_xor_u128(tq, o);
        wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
        if (RES) {
            tqr += __shfl_xor_sync(0xffffffffu, tqr, o);
            tf += __shfl_xor_sync(0xffffffffu, tf, o);
        }
    }
    if (lane == 0) { s_q[warp] = tq; s_qr[warp] = tqr; s_f[warp] = tf; s_w[warp] = wsum; }
    __syncthreads();
    if (warp == 0) {  // the totals by shuffles; thread 0 then builds the header
        u128 T = s_q[lane];
        uint64_t Tr = RES ? s_qr[lane] : 0;
        int64_t F = RES ? s_f[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            T += shfl_xor_u128(T, o);
            if (RES) {
                Tr += __shfl_xor_sync(0xffffffffu, Tr, o);
                F += __shfl_xor_sync(0xffffffffu, F, o);
            }
        }
        const uint64_t x = s_w[lane];  // exclusive prefix of the warps' chunks
        const uint64_t inc = warp_inclusive_sum(x);
        s_w[lane] = inc - x;
        if (lane == 0) {
            h->qoff = 0;
            int ok = (st0 == 0);
            if (T < (u128)T_LO || T > (u128)T_HI) { raise_status(status, SMC_EUNNORMALIZED); ok = 0; }
            int64_t M = (int64_t)m_out;
            uint64_t Tm = (uint64_t)T;
            if (ok && RES && n > 1) {
                M = (int64_t)m_out - F;
                if (M < 0) { raise_status(status, SMC_EUNNORMALIZED); ok = 0; }
                if (M > 0 && Tr == 0) { raise_status(status, SMC_EUNNORMALIZED); ok = 0; }
                Tm = Tr;
            }
            int64_t draws = 0;
            if (n > 1 && M > 0) draws = is_systematic(scheme) ? 1 : M;
            if (ok && u && n_u < draws) { raise_status(status, SMC_EUNIFORMS); ok = 0; }
            h->T = (uint64_t)T;
            h->Tm = Tm;
            h->M = (uint64_t)(M > 0 ? M : 0);
            h->ratio = Tm ? (double)(M > 0 ? M : 0) / (double)Tm : 0.0;
            h->guard = (double)(M > 0 ? M : 1) * 7.105427357601002e-15;
            h->draws = draws;
            h->trivial = (n == 1);
            h->Z_total = h->S_total = h->P_total = 0;
            if (ok) {
                h->c0 = c00;
                if (!u) *ctr = c00 + (uint64_t)draws;
                if (is_systematic(scheme))
                    h->m_sys = draws ? (u ? (uint64_t)(u[0] * TWO53) : draw53(c00, stream, key)) : 0;
            }
            h->active = ok;
            h->mn_direct = 0;
            h->mn_rb = Tm ? ldexp(1.0, L.mg.kb) / (double)Tm : 0.0;
            s_ok = ok;
        }
    }
    if (is_multinomial(scheme)) {  // the multinomial bins: empty, every start at the last particle
        const MnGeom g = L.mg;  // host-computed (Layout)
        for (int64_t b = threadIdx.x; b <= g.nb; b += SB) {
            L.mn_fill[b] = 0;
            L.mn_start[b] = (uint32_t)(n - 1);
        }
    }
    __syncthreads();
    if (!s_ok) return;
    uint64_t carry = s_w[warp];  // (qoff = 0 on one GPU)
#pragma unroll
    for (int k = 0; k < KS; ++k) {
        const int64_t b = w0 + 32 * k + lane;
        const uint64_t inc = warp_inclusive_sum(v[k]);
        if (b < w1) L.tile_pre[b] = carry + inc - v[k];
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
}

// ---------------------------------------------- multinomial / residual (M) --
// Materialize the inclusive CDF Q (or Q') so each draw can binary-search it.
__global__ void __launch_bounds__(RT) k_rs_prefix(int scheme, WSrc src, int64_t n, double m_out, double rscale,
                                                  Layout L)
{
    SMC_PDL_WAIT();
    if (!L.hdr->active || L.hdr->trivial) return;
    if (!mn2_fits(n)) {  // MN1: zero the bin counters (mn1_bins <= n / 256 + 1 <= nt * RT)
        const int64_t b = (int64_t)blockIdx.x * RT + threadIdx.x;
        if (b <= mn1_bins(n)) L.mn_cnt[b] = 0;
    }
    if (L.hdr->M == 0) return;
    __shared__ uint64_t sm[RT / 32 + 1];
    __shared__ uint64_t s_io[tile_smem_elems<uint64_t, RT, RI>()];
    const int64_t tbase = (int64_t)blockIdx.x * TILE;
    uint64_t v[RI];
    // q (or q') from pass A, scanned in place into Q: blocked per thread, moved as whole
    // 32-byte sectors (256-bit loads / stores on full tiles, a shared-memory transpose otherwise)
    load_blocked<RT, RI, uint64_t>(L.qfull, tbase, n, v, s_io, 0ull);
    uint64_t loc = 0;
#pragma unroll
    for (int j = 0; j < RI; ++j) loc += v[j];
    uint64_t tot;
    uint64_t run = L.tile_pre[blockIdx.x] + block_exclusive_sum<RT, uint64_t>(loc, sm, &tot);
    // the multinomial bins' first particles: particle i is the first reached by bin b's
    // positions iff lo_b = floor(b Tm / 2^kb) lies in [Q_{i-1}, Q_i) -- found from the two
    // ends of each particle's interval (ceil bin boundaries are monotone: usually no bin)
    const RsHeader *h = L.hdr;
    const MnGeom g = L.mg;  // host-computed (Layout)
    auto ceil_bin = [&](uint64_t X) {  // min b with floor(b Tm / 2^kb) >= X
        int64_t b = (int64_t)ceil((double)X * h->mn_rb);
        b = b < 0 ? 0 : (b > g.nb ? g.nb : b);
        while (b > 0 && (uint64_t)(((u128)(b - 1) * h->Tm) >> g.kb) >= X) --b;
        while (b < g.nb && (uint64_t)(((u128)b * h->Tm) >> g.kb) < X) ++b;
        return b;
    };
    const int64_t i0 = tbase + (int64_t)threadIdx.x * RI;
    const uint64_t q0 = run;  // Q before this thread's first particle
#pragma unroll
    for (int j = 0; j < RI; ++j) {
        run += v[j];
        v[j] = run;
    }
    if (i0 == 0 && h->qoff > 0) {  // the bin straddling this shard's start reaches particle 0 first
        const int64_t bq = ceil_bin(h->qoff) - 1;
        SMC_CHECK(bq < L.mg.nb + 2);
        if (bq >= 0) L.mn_start[bq] = 0;
    }
    if (i0 < n) {
        // a bin boundary inside this thread's 8 intervals is rare (~8 per 8192 particles): two
        // boundary evaluations per thread, the per-particle walk only when they differ
        int64_t bprev = ceil_bin(q0);
        if (ceil_bin(run) > bprev) {
            uint64_t qprev = q0;
#pragma unroll
            for (int j = 0; j < RI; ++j) {
                if (v[j] > qprev && i0 + j < n) {
                    const int64_t bj = ceil_bin(v[j]);
                    SMC_CHECK(bj <= L.mg.nb + 1);
                    for (int64_t b = bprev; b < bj; ++b) L.mn_start[b] = (uint32_t)(i0 + j);
                    bprev = bj;
                }
                qprev = v[j];
            }
        }
    }
    store_blocked<RT, RI, uint64_t>(L.qfull, tbase, n, v, s_io);
}

// Multinomial positions P_k = floor(m_k Tm / 2^53) (A.3) are iid over the whole CDF: a
// per-draw search over Q diverges across a warp at every level, and a per-draw scatter
// or histogram increment costs a random 32-byte sector each.  Instead:
//  k_mn2_scatter: a block draws 12288 positions into shared memory, counting-sorts them
//      by bin there (bin = the draw's top kb bits), reserves one run per bin in the bin's
//      fixed-capacity region (one global atomic per bin per block), and writes the runs
//      out coalesced (~12 positions = 96 B per bin per block at 2^24);
//  k_mn2_count: one block per bin: the bin's positions reach only the particles
//      [start_b, start_{b+1}] (k_rs_prefix), so their counts accumulate in shared memory
//      (each position found by a search over that slice of Q) and go out with plain
//      coalesced stores -- atomics only for the two end particles a neighbouring bin can
//      share.
// Counts are order-independent integer sums: bit-identical to any other evaluation order.


SMC_DEV uint64_t mn_m(uint64_t k, uint64_t c0, const Key &key, uint64_t stream, const double *u)
{
    return u ? (uint64_t)(u[k] * TWO53) : draw53(c0 + k, stream, key);
}

// DPT draws per thread (mn_dpt): each draw's position and (bin, rank-in-block) stay in
// registers from the drawing pass, the rank being the return of the shared counting atomic, so
// the sort is one pass of direct stores (no second atomic, no permutation array), and the runs'
// global atomics are issued before the block scan and consumed after the sort.
template <int DPT>
__global__ void __launch_bounds__(MT, DPT == 6 ? MN_SCATTER_MINB : 1) k_mn2_scatter(int64_t n, Key key, uint64_t stream, const double *__restrict__ u,
                                                    Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    if (!h->active || h->trivial) return;
    const uint64_t M = h->M, Tm = h->Tm, c0 = h->c0, lo = h->qoff;
    const uint64_t hi = __ldg(&L.qfull[n - 1]);  // inclusive Q (k_rs_prefix): this shard's end
    const MnGeom g = L.mg;  // host-computed (Layout)
    constexpr int mch = MT * DPT;
    const uint64_t k0 = (uint64_t)blockIdx.x * mch;
    if (k0 >= M) return;
    extern __shared__ __align__(16) unsigned char mn_sm[];
    uint64_t *Ps = reinterpret_cast<uint64_t *>(mn_sm);       // the block's positions, sorted by bin
    uint16_t *bs = reinterpret_cast<uint16_t *>(Ps + mch);    // their bins
    uint32_t *hist = reinterpret_cast<uint32_t *>(bs + mch);  // per-bin draw counts of the block
    uint32_t *lofs = hist + g.nb;                             // bin's offset in the block's sorted order
    uint32_t *boff = lofs + g.nb;                             // run start in the bin's region - lofs (mod 2^32)
    __shared__ uint32_t s_w[MT / 32 + 1];
    __shared__ int s_over;
    for (int64_t b = threadIdx.x; b < g.nb; b += MT) hist[b] = 0;
    if (threadIdx.x == 0) s_over = 0;
    __syncthreads();
    const int sh = 53 - g.kb;
    uint64_t P[DPT];
    uint32_t br[DPT];  // (bin << 16) | rank among the block's draws of that bin; ~0 = none
#pragma unroll
    for (int d = 0; d < DPT; ++d) {
        const uint64_t k = k0 + (uint64_t)(d * MT + threadIdx.x);
        br[d] = 0xFFFFFFFFu;
        P[d] = 0;
        if (k < M) {
            const uint64_t m = mn_m(k, c0, key, stream, u);
            const uint64_t p = (uint64_t)(((u128)m * Tm) >> 53);
            if (p >= lo && p < hi) {  // in this shard's slice
                const uint32_t bb = (uint32_t)(m >> sh);
                SMC_CHECK(bb < g.nb);
                P[d] = p;
                br[d] = (bb << 16) | atomicAdd(&hist[bb], 1u);  // rank < mch <= 2^16
            }
        }
    }
    __syncthreads();
    // per bin: the block's run in the bin's region (one global atomic, its result consumed only
    // after the sort), and the bins' offsets in the block's sorted order (exclusive scan over the
    // nb <= 4096 bins, 4 per thread)
    constexpr int BPT = 4;
    uint32_t loc[BPT], rg[BPT], lq[BPT], sum = 0;
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int64_t b = (int64_t)threadIdx.x * BPT + q;
        loc[q] = b < g.nb ? hist[b] : 0;
        sum += loc[q];
        rg[q] = (b < g.nb && loc[q]) ? atomicAdd(&L.mn_fill[b], loc[q]) : 0u;
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_sum<MT, uint32_t>(sum, s_w, &tot);
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int64_t b = (int64_t)threadIdx.x * BPT + q;
        lq[q] = ex;
        if (b < g.nb) lofs[b] = ex;
        ex += loc[q];
    }
    __syncthreads();
#pragma unroll
    for (int d = 0; d < DPT; ++d) {  // the sort: every draw straight to its slot
        if (br[d] != 0xFFFFFFFFu) {
            const uint32_t bb = br[d] >> 16;
            const uint32_t j = lofs[bb] + (br[d] & 0xFFFFu);
            SMC_CHECK(j < (uint32_t)mch);
            Ps[j] = P[d];
            bs[j] = (uint16_t)bb;
        }
    }
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int64_t b = (int64_t)threadIdx.x * BPT + q;
        if (b < g.nb && loc[q]) {
            boff[b] = rg[q] - lq[q];
            if ((uint64_t)rg[q] + loc[q] > (uint64_t)g.cap) s_over = 1;
        }
    }
    __syncthreads();
    if (s_over) {  // a bin overflowed (adversarial uniforms): the direct search handles the call
        if (threadIdx.x == 0) L.hdr_w()->mn_direct = 1;
        return;
    }
    for (uint32_t j = threadIdx.x; j < tot; j += MT) {  // consecutive j: consecutive slots of a bin's run
        const uint32_t bb = bs[j];
        const uint32_t slot = boff[bb] + j;
        SMC_CHECK(bb < g.nb && slot < (uint64_t)g.cap);
        L.mn_pos[(int64_t)bb * g.cap + slot] = Ps[j];
    }
}

// One block per bin: the bin's positions [lo_b, hi_b] are counting-sorted in shared memory
// into NSB sub-buckets of equal width (~1 position each), and every particle of the bin's range
// [start_b, start_{b+1}] counts the positions in its interval [Q_{i-1}, Q_i): whole sub-buckets
// from the sub-bucket prefix, the two end sub-buckets element by element -- O(1) per particle
// and per position, no search.  Interior particles are reached by this bin only (plain
// coalesced stores); the two end particles may be shared with a neighbour (atomics).

// MTC threads: 512 (two blocks per SM) while a bin's shared memory allows it (N <= 2^25), else
// 1024 (same-box A/B, profiles/r2_resample_ab.txt)
template <int MTC, bool ADD>  // ADD: residual -- the counts add onto the floors f_i pass A left in the buffer
__global__ void __launch_bounds__(MTC, 1024 / MTC) k_mn2_count(int64_t n, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    const int64_t b = blockIdx.x;
    // the block's whole first round trip at once: header, fill, the bin's particle range, and
    // (below) the first particle steps' Q -- none depends on another (indices clamped: an inactive
    // call leaves the bin starts unwritten)
    const int32_t active = h->active, trivial = h->trivial, direct = h->mn_direct;
    const uint64_t Tm = h->Tm, qoff = h->qoff;
    const uint32_t fill = __ldg(&L.mn_fill[b]);
    const int64_t s = min((int64_t)__ldg(&L.mn_start[b]), n - 1);
    int64_t e = min(max(s, (int64_t)__ldg(&L.mn_start[b + 1])), n - 1);
    const int64_t e0 = e;
    const uint64_t *Q = L.qfull;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // the bin's particles [s, e] in contiguous per-warp chunks of whole 32-particle steps: a
    // particle's F(Q_{i-1}) is its left neighbour's F(Q_i) (shuffle; across steps, the carry)
    constexpr int PU = 4;  // steps of a warp with their Q loads in flight together
    int64_t c0, c1;
    auto chunk = [&](int64_t last) {
        const int64_t C = (((last - s + 1) + 32 * (MTC / 32) - 1) / (32 * (MTC / 32))) * 32;
        c0 = min(s + warp * C, last + 1);
        c1 = min(c0 + C, last + 1);
    };
    uint64_t q[PU], qfirst = 0;
    int32_t fl[PU];  // residual: the floors f_i already in the histogram buffer, loaded with Q
    auto load_q = [&](int64_t i00) {
#pragma unroll
        for (int k = 0; k < PU; ++k) {
            const int64_t i = i00 + 32 * k + lane;
            q[k] = i < c1 ? __ldg(&Q[i]) : 0;
            fl[k] = ADD && i < c1 ? L.cnt[i] : 0;
        }
    };
    chunk(e);
    load_q(c0);
    if (lane == 0 && c0 < c1) qfirst = c0 ? __ldg(&Q[c0 - 1]) : qoff;
    if (!active || trivial || direct) return;
    const MnGeom g = L.mg;  // host-computed (Layout)
    const int64_t cnt = min((int64_t)fill, g.cap);
    if (cnt == 0) return;
    const uint64_t lo_b = (uint64_t)(((u128)b * Tm) >> g.kb);
    const uint64_t mmax = ((uint64_t)(b + 1) << (53 - g.kb)) - 1;
    const uint64_t hi_b = (uint64_t)(((u128)mmax * Tm) >> 53);  // the bin's largest position
    const uint64_t span = hi_b - lo_b;
    // sub-buckets: a power of two 2^lt >= cnt / 2 (64 .. NSB), so ~2 positions each whatever the
    // draw count (a residual's few remainder draws scan a short prefix); the smallest sh2 with
    // span >> sh2 < 2^lt (one clz, not a loop)
    const int lt = min(12, max(6, 32 - __clz((int)max((int64_t)1, cnt / 2) - 1)));
    static_assert(NSB == 1 << 12, "lt <= 12");
    int sh2 = span ? max(0, 64 - __clzll((long long)span) - lt) : 0;
    while ((span >> sh2) >= ((uint64_t)1 << lt)) ++sh2;
    const int nsb = (int)(span >> sh2) + 1;
    extern __shared__ __align__(16) unsigned char c_sm[];
    uint64_t *Ps = reinterpret_cast<uint64_t *>(c_sm);                 // positions sorted by sub-bucket
    uint32_t *offs = reinterpret_cast<uint32_t *>(Ps + g.cap);         // sub-bucket starts (nsb + 1)
    uint32_t *cur = offs + NSB + 1;                                    // counts, then cursors
    __shared__ uint32_t s_w[MTC / 32 + 1];
    for (int k = threadIdx.x; k <= nsb; k += MTC) cur[k] = 0;
    __syncthreads();
    const uint64_t *pos = L.mn_pos + b * g.cap;
    // up to KPT positions per thread stay in registers with their rank in their sub-bucket (the
    // counting atomic's return value): one read of the bin and no second atomic; larger bins
    // (N > 2^25: wider bins) read their positions twice
    constexpr int KPT = 8;
    const bool inreg = cnt <= (int64_t)MTC * KPT;
    uint64_t Pr[KPT];
    uint32_t sbr[KPT];
    if (inreg) {
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
            const int64_t j = threadIdx.x + (int64_t)k * MTC;
            Pr[k] = j < cnt ? pos[j] : 0;
        }
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
            const int64_t j = threadIdx.x + (int64_t)k * MTC;
            if (j < cnt) {
                const uint32_t sb = (uint32_t)((Pr[k] - lo_b) >> sh2);
                SMC_CHECK(sb < (uint32_t)nsb);
                sbr[k] = (sb << 16) | atomicAdd(&cur[sb], 1u);  // rank < 2^16: cnt <= MTC * KPT
            }
        }
    } else {
        for (int64_t j = threadIdx.x; j < cnt; j += MTC) atomicAdd(&cur[(pos[j] - lo_b) >> sh2], 1u);
    }
    __syncthreads();
    {  // exclusive scan of the nsb <= NSB sub-bucket counts, 4 per thread
        constexpr int SPT = NSB / MTC;
        uint32_t c8[SPT], sum = 0;
#pragma unroll
        for (int k8 = 0; k8 < SPT; ++k8) {
            const int k = threadIdx.x * SPT + k8;
            c8[k8] = k < nsb ? cur[k] : 0;
            sum += c8[k8];
        }
        uint32_t tot;
        uint32_t ex = block_exclusive_sum<MTC, uint32_t>(sum, s_w, &tot);
#pragma unroll
        for (int k8 = 0; k8 < SPT; ++k8) {
            const int k = threadIdx.x * SPT + k8;
            if (k < nsb) { offs[k] = ex; cur[k] = ex; }
            ex += c8[k8];
        }
        if (threadIdx.x == 0) offs[nsb] = tot;
    }
    __syncthreads();
    if (inreg) {
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
            const int64_t j = threadIdx.x + (int64_t)k * MTC;
            SMC_CHECK(j >= cnt || offs[sbr[k] >> 16] + (sbr[k] & 0xFFFFu) < (uint64_t)g.cap);
            if (j < cnt) Ps[offs[sbr[k] >> 16] + (sbr[k] & 0xFFFFu)] = Pr[k];
        }
    } else {
        for (int64_t j = threadIdx.x; j < cnt; j += MTC) {  // the bin's positions again (L2-hot): placed
            const uint64_t P = pos[j];
            Ps[atomicAdd(&cur[(P - lo_b) >> sh2], 1u)] = P;
        }
    }
    __syncthreads();
    if (e == n - 1) {  // the start sentinel (the last bin, or zero-weight particles to the end):
        __shared__ int64_t s_e;  // the particle of the bin's largest position instead, by search
        if (threadIdx.x == 0) {
            const uint64_t Pm = min(hi_b, __ldg(&Q[n - 1]) - 1);
            int64_t lo = s, hi = n - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (__ldg(&Q[mid]) > Pm) hi = mid; else lo = mid + 1;
            }
            s_e = lo;
        }
        __syncthreads();
        e = s_e;
    }
    // F(X) = #{bin positions < X}: the sub-bucket prefix plus the few positions of X's own
    // sub-bucket below X; particle i's count is F(Q_i) - F(Q_{i-1}), the second term being the
    // previous particle's first (the neighbouring lane's, by shuffle)
    auto F = [&](uint64_t X) -> uint32_t {
        if (X <= lo_b) return 0;
        if (X > hi_b) return offs[nsb];
        const int sb = (int)((X - lo_b) >> sh2);
        const uint32_t a = offs[sb], z = offs[sb + 1];
        uint32_t c = a;
        // the sub-bucket's first MN_FU positions predicated, not looped: a warp no longer runs
        // its lanes' longest scan (~6 for ~2 positions per sub-bucket) iteration by iteration;
        // the rare remainder loops
#pragma unroll
        for (int t = 0; t < MN_FU; ++t) c += (a + t < z && Ps[a + t] < X) ? 1u : 0u;
        for (uint32_t k = a + MN_FU; k < z; ++k) c += (Ps[k] < X);
        return c;
    };
    if (e != e0) {  // the sentinel search moved the end: re-chunk (the last bin only)
        chunk(e);
        load_q(c0);
        if (lane == 0 && c0 < c1) qfirst = c0 ? __ldg(&Q[c0 - 1]) : qoff;
    }
    uint32_t carry = lane == 0 && c0 < c1 ? F(qfirst) : 0;  // F(Q_{c0-1}), lane 0's left neighbour
    for (int64_t i00 = c0; i00 < c1; i00 += 32 * PU) {
        if (i00 != c0) load_q(i00);  // the first steps' Q came with the header
#pragma unroll
        for (int k = 0; k < PU; ++k) {
            const int64_t i = i00 + 32 * k + lane;
            const uint32_t Fi = i < c1 ? F(q[k]) : 0;
            uint32_t Fp = __shfl_up_sync(0xffffffffu, Fi, 1);
            if (lane == 0) Fp = carry;
            carry = __shfl_sync(0xffffffffu, Fi, 31);
            if (i >= c1) continue;
            const uint32_t c = Fi - Fp;
            SMC_CHECK(i >= 0 && i < n);
            if (i == s || i == e) {  // a neighbouring bin may reach it too
                if (c) atomicAdd(&L.cnt[i], (int)c);
            } else {
                L.cnt[i] = fl[k] + (int32_t)c;  // only this bin reaches it (+ f_i: residual)
            }
        }
    }
}

// ---- MN1: the multinomial path for N past mn2_fits (round 1's; every draw regenerated from its
// counter in two passes).  Draws COUNTED then SCATTERED into ~256-particle position bins in
// global memory (bin = an arithmetic, monotone function of P), each bucketed position then
// searched between its bin's first particles: a warp's 32 searches share their paths down to
// the last few levels.  Counts are order-independent integer sums: bit-identical to MN2.
struct Mn1Ctx {
    uint64_t M, Tm, c0, lo, hi;  // [lo, hi): this shard's slice of the CDF
    uint32_t nb;
    uint64_t W;                  // bin width: bin b = positions [lo + b W, lo + (b+1) W)
    double invW;
    SMC_DEV uint32_t bin(uint64_t P) const  // exact floor((P - lo) / W)
    {
        const uint64_t d = P - lo;
        uint64_t b = (uint64_t)((double)d * invW);
        while (b && b * W > d) --b;
        while ((b + 1) * W <= d) ++b;
        return (uint32_t)(b < nb ? b : nb - 1);
    }
};

SMC_DEV Mn1Ctx mn1_ctx(const Layout &L, int64_t n)
{
    const RsHeader *h = L.hdr;
    Mn1Ctx c;
    c.M = h->M;
    c.Tm = h->Tm;
    c.c0 = h->c0;
    c.lo = h->qoff;
    c.hi = __ldg(&L.qfull[n - 1]);  // inclusive Q (k_rs_prefix): this shard's end
    c.nb = (uint32_t)mn1_bins(n);
    const uint64_t span = c.hi > c.lo ? c.hi - c.lo : 1;
    c.W = span / c.nb + 1;  // nb W > span: every position has a bin
    c.invW = 1.0 / (double)c.W;
    return c;
}

SMC_DEV uint64_t mn1_position(const Mn1Ctx &c, uint64_t k, const Key &key, uint64_t stream, const double *u)
{
    const uint64_t m = u ? (uint64_t)(u[k] * TWO53) : draw53(c.c0 + k, stream, key);
    return (uint64_t)(((u128)m * c.Tm) >> 53);
}

// atomicAdd(&a[key], 1) for a warp, one atomic when every active lane shares the key
// (degenerate weights send every draw to one bin / one particle: without this the
// same-address atomics serialize).  Returns the lane's slot (old value + rank).
SMC_DEV uint32_t agg_inc(uint32_t *a, uint32_t key, bool active)
{
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (!act) return 0;
    const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
    const uint32_t k0 = __shfl_sync(0xffffffffu, key, leader);
    if (__all_sync(0xffffffffu, !active || key == k0)) {  // the whole warp hits one counter
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&a[k0], (uint32_t)__popc(act));
        base = __shfl_sync(0xffffffffu, base, leader);
        return base + __popc(act & ((1u << lane) - 1));
    }
    return active ? atomicAdd(&a[key], 1u) : 0;
}

__global__ void k_mn1_count(int64_t n, Key key, uint64_t stream, const double *__restrict__ u, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    if (!h->active || h->trivial) return;
    const Mn1Ctx c = mn1_ctx(L, n);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t kend = (c.M + stride - 1) / stride * stride;  // whole warps iterate together
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < kend; k += stride) {
        const uint64_t P = k < c.M ? mn1_position(c, k, key, stream, u) : c.lo;
        const bool in = k < c.M && P >= c.lo && P < c.hi;  // else: past the end, or on another shard
        agg_inc(L.mn_cnt, in ? c.bin(P) : 0u, in);
    }
}

// one block: exclusive bucket offsets; fill pointers back to zero
__global__ void __launch_bounds__(SB) k_mn1_scan(int64_t nbins, int64_t cap, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    if (!h->active || h->trivial) return;
    __shared__ uint64_t sm64[SB / 32 + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = SB / 32;
    const int64_t nt = nbins;
    const int64_t C = (nt + NW - 1) / NW;
    const int64_t w0 = warp * C < nt ? warp * C : nt, w1 = w0 + C < nt ? w0 + C : nt;
    constexpr int KS = 8;  // warp-rows of bins in flight per round (one round trip per round)
    uint64_t wsum = 0;
    for (int64_t b0 = w0 + lane; b0 < w1; b0 += 32 * KS) {
        uint32_t v[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) v[k] = b0 + 32 * k < w1 ? L.mn_cnt[b0 + 32 * k] : 0;
#pragma unroll
        for (int k = 0; k < KS; ++k) wsum += v[k];
    }
    wsum = warp_sum(wsum);
    if (lane == 0) sm64[warp] = wsum;
    __syncthreads();
    if (warp == 0) {
        const uint64_t x = sm64[lane];
        const uint64_t inc = warp_inclusive_sum(x);
        sm64[lane] = inc - x;
    }
    __syncthreads();
    uint64_t carry = sm64[warp];
    for (int64_t c0 = w0; c0 < w1; c0 += 32 * KS) {
        uint64_t vv[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) vv[k] = c0 + 32 * k + lane < w1 ? L.mn_cnt[c0 + 32 * k + lane] : 0;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            const int64_t b = c0 + 32 * k + lane;
            const uint64_t inc = warp_inclusive_sum(vv[k]);
            if (b < w1) {
                L.mn_off[b] = (uint32_t)(carry + inc - vv[k]);
                L.mn_fill[b] = 0;
            }
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    if (warp == NW - 1 && lane == 31) {
        L.mn_off[nt] = (uint32_t)carry;  // total positions in this shard
        L.hdr->mn_direct = carry > (uint64_t)cap;  // buckets hold `cap` positions
    }
}

// first particle of every bin: mn_start[b] = first i with Q_i > lo + b W (b = 0..nb)
__global__ void k_mn1_starts(int64_t n, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    if (!h->active || h->trivial || h->mn_direct) return;
    const Mn1Ctx c = mn1_ctx(L, n);
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= c.nb; b += gridDim.x * blockDim.x) {
        const uint64_t X = c.lo + (uint64_t)b * c.W;
        int64_t lo = 0, hi = n - 1;
        if (X >= c.hi) lo = n - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(&L.qfull[mid]) > X) hi = mid; else lo = mid + 1;
        }
        L.mn_start[b] = (uint32_t)lo;
    }
}

__global__ void k_mn1_scatter(int64_t n, Key key, uint64_t stream, const double *__restrict__ u, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    if (!h->active || h->trivial) return;
    if (h->mn_direct) return;  // more positions than bucket capacity (a shard): k_rs_multinomial
    const Mn1Ctx c = mn1_ctx(L, n);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t kend = (c.M + stride - 1) / stride * stride;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < kend; k += stride) {
        const uint64_t P = k < c.M ? mn1_position(c, k, key, stream, u) : c.lo;
        const bool in = k < c.M && P >= c.lo && P < c.hi;
        const uint32_t b = in ? c.bin(P) : 0u;
        const uint32_t r = agg_inc(L.mn_fill, b, in);
        SMC_CHECK(!in || (b < c.nb && __ldg(&L.mn_off[b]) + r < (uint64_t)n));
        if (in) L.mn_pos[__ldg(&L.mn_off[b]) + r] = P;
    }
}

// per bucketed position: first i with Q_i > P (Q inclusive, materialized by k_rs_prefix),
// searched only between its bin's first particles
__global__ void k_mn1_assign(int64_t n, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    if (!h->active || h->trivial) return;
    if (h->mn_direct) return;
    const Mn1Ctx c = mn1_ctx(L, n);
    const uint32_t total = __ldg(&L.mn_off[mn1_bins(n)]);
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t jend = (total + stride - 1) / stride * stride;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < jend; j += stride) {
        const bool in = j < total;
        int64_t lo = 0;
        if (in) {
            const uint64_t P = L.mn_pos[j];
            const uint32_t b = c.bin(P);
            SMC_CHECK(b < c.nb);
            lo = __ldg(&L.mn_start[b]);
            int64_t hi = __ldg(&L.mn_start[b + 1]);
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (__ldg(&L.qfull[mid]) > P) hi = mid; else lo = mid + 1;
            }
        }
        agg_inc(reinterpret_cast<uint32_t *>(L.cnt), (uint32_t)lo, in);
    }
}

// Direct fallback (a shard receiving more draws than its bucket capacity): per draw,
// binary search over this shard's whole Q.
__global__ void k_rs_multinomial(int64_t n, Key key, uint64_t stream, const double *__restrict__ u, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    if (!h->active || h->trivial || !h->mn_direct) return;
    const uint64_t M = h->M, Tm = h->Tm, c0 = h->c0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < M; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t m = u ? (uint64_t)(u[k] * TWO53) : draw53(c0 + k, stream, key);
        const uint64_t P = (uint64_t)(((u128)m * Tm) >> 53);
        if (P < h->qoff || P >= __ldg(&L.qfull[n - 1])) continue;  // position on another shard
        int64_t lo = 0, hi = n - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(&L.qfull[mid]) > P) hi = mid; else lo = mid + 1;
        }
        atomicAdd(&L.cnt[lo], 1);
    }
}

// ------------------------------------------------------------------ pass B --
struct StratCtx {
    uint64_t Tm, M, m_sys, c0, stream;
    double ratio, guard;
    const double *u;
    Key key;
    bool systematic;
    bool force;     // test hook g_force_exact, read once per thread
    double us_sys;  // m_sys 2^-53 (systematic)
};

template <bool SYS>
SMC_DEV uint64_t m_of(const StratCtx &c, uint64_t s)
{
    if (SYS) return c.m_sys;
    if (c.u) return (uint64_t)(c.u[s] * TWO53);
    return draw53(c.c0 + s, c.stream, c.key);
}

// Exact F(X) = #{k < M : P_k < X},  P_k = floor((k 2^53 + m_k) Tm / (M 2^53)):
// k < s := floor(X M / Tm) all qualify, k > s none; k = s iff m_s Tm < (X M - s Tm) 2^53.
template <bool SYS>
SMC_DEV uint64_t F_exact(const StratCtx &c, uint64_t X)
{
    if (X >= c.Tm) return c.M;
    if (X == 0) return 0;
    const u128 XM = (u128)X * c.M;
    uint64_t s = (uint64_t)((double)X * c.ratio);
    while ((u128)s * c.Tm > XM) --s;
    while ((u128)(s + 1) * c.Tm <= XM) ++s;
    const u128 rem = XM - (u128)s * c.Tm;
    const uint64_t m = m_of<SYS>(c, s);
    return s + (((u128)m * c.Tm < (rem << 53)) ? 1 : 0);
}

// Same value in ~10 instructions: z = X M / Tm in fp64 (|error| <= 3.4e-16 M);
// F = floor(z) + [u_s < frac(z)].  Whenever frac(z) or frac(z) - u_s lies
// inside the guard band the exact path decides, so the result is bit-identical.
template <bool SYS>
SMC_DEV uint64_t F_fast(const StratCtx &c, uint64_t X)
{
    if (X >= c.Tm) return c.M;
    const double z = (double)X * c.ratio;
    const double fl = floor(z);
    const double fr = z - fl;
    const uint64_t s = (uint64_t)fl;
    const double us = SYS ? c.us_sys : (double)m_of<SYS>(c, s) * INV53;
    const double d = fr - us;
    // |fr - 1/2| > 1/2 - guard  <=>  fr < guard or fr > 1 - guard (X == 0 lands here too)
    if (c.force || fabs(fr - 0.5) > 0.5 - c.guard || fabs(d) < c.guard) return F_exact<SYS>(c, X);
    return s + (d > 0.0 ? 1 : 0);
}

// F_fast without its branch: the fast value, and `ex` set when the exact path must decide
// (X >= Tm, X == 0 or a guard-band hit) -- per-element loops stay branch-free and fall
// back warp-wide only when some lane needs it.
template <bool SYS>
SMC_DEV uint64_t F_fast_flag(const StratCtx &c, uint64_t X, bool &ex)
{
    // (a conversion-free variant -- X and floor(z) through the 2^52 shifter -- measured slower:
    // 12 fp64 operations per item instead of 3 conversions, the same pipe time, more issue slots)
    const double z = (double)X * c.ratio;
    const double fl = floor(z);
    const double fr = z - fl;
    const uint64_t s = (uint64_t)fl;
    const double us = SYS ? c.us_sys : (double)m_of<SYS>(c, s < c.M ? s : c.M - 1) * INV53;
    const double d = fr - us;
    ex = c.force || X >= c.Tm || fabs(fr - 0.5) > 0.5 - c.guard || fabs(d) < c.guard;
    return s + (d > 0.0 ? 1 : 0);
}

// pack (zero slots, surplus parents) in the top 2 x 14 bits, surplus children in
// the low 36 -- tile-local sums never carry across fields (<= 2048, < 2^31).
SMC_DEV uint64_t pack_zsp(uint32_t z, uint32_t p, uint64_t s) { return ((uint64_t)z << 50) | ((uint64_t)p << 36) | s; }
SMC_DEV uint32_t unz(uint64_t v) { return (uint32_t)(v >> 50); }
SMC_DEV uint32_t unp(uint64_t v) { return (uint32_t)((v >> 36) & 0x3FFF); }
SMC_DEV uint64_t uns(uint64_t v) { return v & ((1ull << 36) - 1); }

// blocked smem index with one pad word per 16: conflict-free for 64-bit reads of t*8+j
SMC_DEV int pad16(int i) { return i + (i >> 4); }

// replication_to_parents' rank scan as REDUCE-THEN-SCAN over
// 2048-slot tiles: (1) the pass that holds a tile's counts publishes its
// (zero slots, surplus parents, surplus children) aggregate; (2) one block scans
// the aggregates (k_rs_zsp_scan); (3) k_rs_ranks re-reads the counts and emits
// the compacted surplus-parent list.  (A decoupled lookback fused into pass B1
// was measured slower on B200: the status chain over 8192 tiles costs more than
// the 4 B/slot re-read -- DESIGN.md §6.)
SMC_DEV void tile_aggregate(const int32_t (&c)[RI], int64_t b, const Layout &L)
{
    __shared__ uint64_t sm[RT / 32 + 1];
    uint32_t tz = 0, tp = 0;
    uint64_t ts = 0;
#pragma unroll
    for (int j = 0; j < RI; ++j) {
        tz += (c[j] == 0);
        tp += (c[j] >= 2);
        ts += c[j] >= 2 ? (uint64_t)(c[j] - 1) : 0;
    }
    uint64_t agg;
    block_exclusive_sum<RT, uint64_t>(pack_zsp(tz, tp, ts), sm, &agg);
    if (threadIdx.x == 0) L.tile_zsp[b] = agg;
}

// The tile's zero-count slots as a bitmask: thread t's RI = 8 slots are byte t, four threads per
// 32-bit word, 64 words per tile (one coalesced 256-byte store).  Padding slots hold 1: not zero.
SMC_DEV void zero_mask(const int32_t (&c)[RI], int64_t b, const Layout &L)
{
    static_assert(RI == 8, "one byte of zero flags per thread");
    uint32_t zb = 0;
#pragma unroll
    for (int j = 0; j < RI; ++j) zb |= (uint32_t)(c[j] == 0) << j;
    const int lane = threadIdx.x & 31;
    uint32_t wv = zb << (8 * (lane & 3));
    wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
    wv |= __shfl_xor_sync(0xffffffffu, wv, 2);
    if ((lane & 3) == 0) L.zmask[b * (TILE / 32) + (threadIdx.x >> 2)] = wv;
}

// One block: exclusive (Z, S, P) prefix of the tile aggregates, the totals, each
// slot tile's first zero rank, and the sum(counts) == N check.
__global__ void __launch_bounds__(SB) k_rs_zsp_scan(int64_t nt, int whole, int32_t *status, Layout L)
{
    SMC_PDL_WAIT();
    RsHeader *h = L.hdr;
    __shared__ uint64_t s_zp[SB / 32 + 1], s_s[SB / 32 + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = SB / 32;
    const int64_t C = (nt + NW - 1) / NW;  // warp w owns tiles [w C, (w+1) C)
    const int64_t w0 = warp * C < nt ? warp * C : nt, w1 = w0 + C < nt ? w0 + C : nt;
    // (Z, P) as two 32-bit halves of one u64 (totals < 2^31 never carry), S as u64
    auto zp = [&](uint64_t v) { return ((uint64_t)unz(v) << 32) | unp(v); };
    constexpr int KS = 8;  // warp-rows of tiles in flight per round (one round trip per round)
    // nt <= 8 SB (N <= 2^24): the first round's loads are all of them, kept for the scan; they are
    // issued together with the header's flags (the aggregates are valid workspace either way)
    const bool one = C <= 32 * KS;
    uint64_t v0[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) v0[k] = w0 + lane + 32 * k < w1 ? L.tile_zsp[w0 + lane + 32 * k] : 0;
    if (!h->active || h->trivial) return;
    uint64_t a = 0, bs = 0;
#pragma unroll
    for (int k = 0; k < KS; ++k) { a += zp(v0[k]); bs += uns(v0[k]); }
    for (int64_t t0 = w0 + lane + 32 * KS; t0 < w1; t0 += 32 * KS) {
        uint64_t v[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) v[k] = t0 + 32 * k < w1 ? L.tile_zsp[t0 + 32 * k] : 0;
#pragma unroll
        for (int k = 0; k < KS; ++k) { a += zp(v[k]); bs += uns(v[k]); }
    }
    a = warp_sum(a);
    bs = warp_sum(bs);
    if (lane == 0) { s_zp[warp] = a; s_s[warp] = bs; }
    __syncthreads();
    if (warp == 0) {
        const uint64_t x = s_zp[lane], y = s_s[lane];
        const uint64_t ix = warp_inclusive_sum(x), iy = warp_inclusive_sum(y);
        s_zp[lane] = ix - x;
        s_s[lane] = iy - y;
        if (lane == 31) {
            const uint32_t Z = (uint32_t)(ix >> 32), P = (uint32_t)ix, S = (uint32_t)iy;
            h->Z_total = Z;
            h->S_total = S;
            h->P_total = P;
            L.sp_start[P] = (int32_t)S;  // sentinel
            L.tile_z0[nt] = (int32_t)Z;
            L.tile_excl[nt] = make_uint4(Z, S, P, 0);
            // sum(counts) != N; a shard's Z and S only balance globally (host check)
            if (whole && Z != S) raise_status(status, SMC_ECOUNTS);
        }
    }
    __syncthreads();
    uint64_t ca = s_zp[warp], cs = s_s[warp];
    auto emit = [&](int64_t c0, const uint64_t(&vv)[KS]) {
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            const int64_t t = c0 + 32 * k + lane;
            const uint64_t x = zp(vv[k]), y = uns(vv[k]);
            const uint64_t ix = warp_inclusive_sum(x), iy = warp_inclusive_sum(y);
            if (t < w1) {
                const uint64_t ex = ca + ix - x, ey = cs + iy - y;
                L.tile_excl[t] = make_uint4((uint32_t)(ex >> 32), (uint32_t)ey, (uint32_t)ex, 0);
                L.tile_z0[t] = (int32_t)(ex >> 32);
            }
            ca += __shfl_sync(0xffffffffu, ix, 31);
            cs += __shfl_sync(0xffffffffu, iy, 31);
        }
    };
    if (one) {
        emit(w0, v0);
        return;
    }
    for (int64_t c0 = w0; c0 < w1; c0 += 32 * KS) {
        uint64_t vv[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) vv[k] = c0 + 32 * k + lane < w1 ? L.tile_zsp[c0 + 32 * k + lane] : 0;
        emit(c0, vv);
    }
}

// Emission for one tile whose exclusive prefix is known: the tile's slice of the
// compacted surplus-parent list (index, first surplus rank) -- staged in shared
// memory and stored coalesced -- and the rank anchors (the surplus parent
// covering every ANCHOR-th surplus rank).
__global__ void __launch_bounds__(RT) k_rs_ranks(const int32_t *__restrict__ cin, int64_t n, int32_t *status,
                                                 int check, Layout L)
{
    SMC_PDL_WAIT();
    RsHeader *h = L.hdr;
    if (!h->active || h->trivial) return;
    __shared__ int32_t s_c[tile_smem_elems<int32_t, RT, RI>()];
    __shared__ int32_t s_stage[2 * TILE];
    __shared__ uint64_t sm[RT / 32 + 1];
    const int64_t b = blockIdx.x;
    int32_t c[RI];
    const uint4 ex = __ldcg(&L.tile_excl[b]);  // issued before the counts' load and scan: its latency overlaps
    load_blocked<RT, RI, int32_t>(cin, b * TILE, n, c, s_c, 1);  // coalesced; pad: not zero, no surplus
    if (check) {  // caller-provided counts (replication_to_parents): the first negative one is reported
#pragma unroll
        for (int j = 0; j < RI; ++j)
            if (c[j] < 0) {
                raise_status_at(status, SMC_ECOUNTS, b * TILE + (int64_t)threadIdx.x * RI + j);
                c[j] = 0;
            }
    }
    uint32_t tp = 0;
    uint64_t ts = 0;
#pragma unroll
    for (int j = 0; j < RI; ++j) {
        tp += (c[j] >= 2);
        ts += c[j] >= 2 ? (uint64_t)(c[j] - 1) : 0;
    }
    uint64_t agg;
    const uint64_t tex = block_exclusive_sum<RT, uint64_t>(pack_zsp(0, tp, ts), sm, &agg);
    uint32_t sr = ex.y + (uint32_t)uns(tex);
    uint32_t lp = unp(tex);  // tile-local surplus-parent index
    const int32_t base = (int32_t)(b * TILE) + (int32_t)threadIdx.x * RI;  // n < 2^31
#pragma unroll
    for (int j = 0; j < RI; ++j) {
        if (c[j] >= 2) {  // padding slots load as 1
            SMC_CHECK(c[j] < 2 || lp < (uint32_t)TILE);
            s_stage[lp] = base + j;
            s_stage[TILE + lp] = (int32_t)sr;
            ++lp;
            sr += (uint32_t)(c[j] - 1);
        }
    }
    __syncthreads();
    const uint32_t np = unp(agg);
    for (uint32_t k = threadIdx.x; k < np; k += RT) {
        SMC_CHECK(ex.z + k <= (uint64_t)n);
        L.sp_idx[ex.z + k] = s_stage[k];
        L.sp_start[ex.z + k] = s_stage[TILE + k];
    }
    // rank anchors: every multiple of ANCHOR in this tile's surplus ranks [ex.y, ex.y + S_tile),
    // spread over the block (a parent with a huge surplus -- degenerate weights -- would
    // otherwise write N/ANCHOR anchors from one thread); owner by search in the staged starts
    // a shard's surplus can exceed its n slots (children leaving for other shards): anchors
    // exist for ranks < (n/ANCHOR + 2) ANCHOR only -- all pass C needs (its ranks are < n);
    // k_rs_pack searches beyond them
    const uint32_t cap_r = (uint32_t)(n / ANCHOR + 2) * ANCHOR;  // the anchor buffer's extent in ranks
    const uint32_t s0 = ex.y, s1 = min(ex.y + (uint32_t)uns(agg), cap_r);
    for (uint32_t a = (s0 + ANCHOR - 1) / ANCHOR + threadIdx.x; a * ANCHOR < s1 && np; a += RT) {
        const uint32_t r = a * ANCHOR;
        uint32_t lo = 0, hi = np;  // last k with start_k <= r
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((uint32_t)s_stage[TILE + mid] <= r) lo = mid; else hi = mid;
        }
        SMC_CHECK(a < (uint32_t)(n / ANCHOR + 2) && lo < np);
        L.anchor[a] = (int32_t)(ex.z + lo);
    }
}

// Aggregates of caller-provided counts (replication_to_parents without pass B1).
__global__ void __launch_bounds__(RT) k_rs_aggs(const int32_t *__restrict__ cin, int64_t n, Layout L)
{
    SMC_PDL_WAIT();
    if (!L.hdr->active || L.hdr->trivial) return;
    __shared__ int32_t s_c[tile_smem_elems<int32_t, RT, RI>()];
    int32_t c[RI];
    load_blocked<RT, RI, int32_t>(cin, (int64_t)blockIdx.x * TILE, n, c, s_c, 1);
#pragma unroll
    for (int j = 0; j < RI; ++j) c[j] = c[j] < 0 ? 0 : c[j];  // k_rs_ranks raises ECOUNTS
    zero_mask(c, blockIdx.x, L);
    tile_aggregate(c, blockIdx.x, L);
}

// Pass B1: counts per particle.  Embarrassingly parallel (no inter-tile wait);
// the counts go to `counts` (the caller's or the workspace's).
template <bool RES, bool MULTI, bool SYS>  // scheme family, resolved at compile time
__global__ void __launch_bounds__(RT, RS_COUNTS_MINB) k_rs_counts(int scheme, WSrc src, int64_t n, double m_out, double rscale,
                                                  Key key, uint64_t stream, const double *__restrict__ u,
                                                  int32_t *__restrict__ counts, int ranks, Layout L)
{
    SMC_PDL_WAIT();
    RsHeader *h = L.hdr;
    if (!h->active) return;
    __shared__ uint64_t sm[RT / 32 + 1];
    __shared__ uint64_t s_q[tile_smem_elems<uint64_t, RT, RI>()];
    __shared__ int32_t s_fb[tile_smem_elems<uint64_t, RT, RI>()];
    if (h->trivial) {  // N == 1: no-op resample
        if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = (int32_t)m_out;
        return;
    }
    const int64_t b = blockIdx.x;
    const int64_t tbase = b * TILE;
    const int64_t base = tbase + (int64_t)threadIdx.x * RI;  // blocked: thread owns RI consecutive
    int32_t c[RI];
    const bool full = tbase + TILE <= n;  // no per-element bounds checks on full tiles
    const uint64_t tpre = MULTI ? 0 : L.tile_pre[b];  // issued before the tile's loads and scan
    {
        uint64_t q[RI];
        int32_t f[RI];
        uint64_t loc = 0;
        // q_i (q'_i for the residual schemes) was materialized by pass A, and the residual floors
        // f_i too (in the histogram buffer): no exp / quantization here, 64 + 32 contiguous bytes
        // per thread (residual-multinomial: the floors are already in the draws' histogram)
        if (!MULTI) {
            load_blocked<RT, RI, uint64_t>(L.qfull, tbase, n, q, s_q, 0ull);  // coalesced
        } else {
#pragma unroll
            for (int j = 0; j < RI; ++j) q[j] = 0;  // multinomial: counts come from the histogram
        }
        if (RES && !MULTI) {
            load_blocked<RT, RI, int32_t>(L.cnt, tbase, n, f, s_fb, 0);
        } else {
#pragma unroll
            for (int j = 0; j < RI; ++j) f[j] = 0;
        }
#pragma unroll
        for (int j = 0; j < RI; ++j) loc += q[j];
        if (MULTI) {
            int32_t h4[RI];
            load_blocked<RT, RI, int32_t>(L.cnt, tbase, n, h4, s_fb, 0);  // the draws' histogram (+ f_i)
#pragma unroll
            for (int j = 0; j < RI; ++j) c[j] = (full || base + j < n) ? f[j] + h4[j] : 1;
        } else {
            uint64_t tot;
            uint64_t X = tpre + block_exclusive_sum<RT, uint64_t>(loc, sm, &tot);
            StratCtx sc;
            sc.Tm = h->Tm;
            sc.M = h->M;
            sc.m_sys = h->m_sys;
            sc.c0 = h->c0;
            sc.ratio = h->ratio;
            sc.guard = h->guard;
            sc.stream = stream;
            sc.u = u;
            sc.key = key;
            sc.systematic = SYS;
            sc.force = g_force_exact != 0;
            sc.us_sys = (double)sc.m_sys * INV53;
            if (sc.M == 0) {  // residual with no leftovers: the floors are the counts
#pragma unroll
                for (int j = 0; j < RI; ++j) c[j] = (full || base + j < n) ? f[j] : 1;
            } else {
                // F at the thread's start and after each of its RI items (padding items have
                // q = 0: F unchanged) by the branch-free fast path; when any lane of the warp
                // flagged an item (rare: the guard band, X = 0 at the very start, X >= Tm at
                // the end) the warp redoes its items with the exact path where flagged
                bool e, any = false;
                uint64_t Xj = X;
                uint64_t Fp = F_fast_flag<SYS>(sc, Xj, e);
                any |= e;
#pragma unroll
                for (int j = 0; j < RI; ++j) {
                    Xj += q[j];
                    const uint64_t Fc = F_fast_flag<SYS>(sc, Xj, e);
                    any |= e;
                    c[j] = (full || base + j < n) ? f[j] + (int32_t)(Fc - Fp) : 1;  // padding: 1
                    Fp = Fc;
                }
                if (__any_sync(0xffffffffu, any)) {  // q re-read from pass A's copy: no indexed registers
                    __shared__ int32_t s_cx[RT * RI];
                    Xj = X;
                    Fp = F_fast<SYS>(sc, Xj);
#pragma unroll 1
                    for (int j = 0; j < RI; ++j) {
                        Xj += (full || base + j < n) ? L.qfull[base + j] : 0;
                        const uint64_t Fc = F_fast<SYS>(sc, Xj);
                        s_cx[threadIdx.x * RI + j] = (int32_t)(Fc - Fp);
                        Fp = Fc;
                    }
#pragma unroll
                    for (int j = 0; j < RI; ++j)
                        if (full || base + j < n) c[j] = f[j] + s_cx[threadIdx.x * RI + j];
                }
            }
        }
    }
    __syncthreads();  // s_fb may still be read by the residual staging path
    store_blocked<RT, RI, int32_t>(counts, tbase, n, c, s_fb);  // coalesced
    if (ranks) {
        zero_mask(c, b, L);   // pass C's zero slots: 1 bit per slot instead of re-reading the counts
        tile_aggregate(c, b, L);  // the parent map's per-tile (Z, S, P) for k_rs_zsp_scan
    }
}

inline void launch_counts(int scheme, unsigned nt, cudaStream_t s, WSrc src, int64_t n, double mo, double rscale,
                          Key key, uint64_t stream, const double *u, int32_t *cout, int ranks, Layout L)
{
#define SMC_COUNTS(R_, M_, S_) \
    smc_launch(k_rs_counts<R_, M_, S_>, nt, RT, 0, s, scheme, src, n, mo, rscale, key, stream, u, cout, ranks, L)
    switch (scheme) {
    case SMC_MULTINOMIAL: SMC_COUNTS(false, true, false); break;
    case SMC_RESIDUAL: SMC_COUNTS(true, true, false); break;
    case SMC_STRATIFIED: SMC_COUNTS(false, false, false); break;
    case SMC_SYSTEMATIC: SMC_COUNTS(false, false, true); break;
    case SMC_RESIDUAL_STRATIFIED: SMC_COUNTS(true, false, false); break;
    default: SMC_COUNTS(true, false, true); break;  // SMC_RESIDUAL_SYSTEMATIC
    }
#undef SMC_COUNTS
}

// ------------------------------------------------------------------ pass C --
SMC_DEV void ld256(const double *p, double4 &v)
{
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
}
SMC_DEV void st256(double *p, const double4 &v)
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}

SMC_DEV void copy_row(char *rows, int64_t row_bytes, int64_t dst, int64_t srcr)
{
    if (row_bytes == 32) {
        double4 v;
        ld256((const double *)(rows + srcr * 32), v);
        st256((double *)(rows + dst * 32), v);
    } else if ((row_bytes & 15) == 0) {
        const int4 *s = (const int4 *)(rows + srcr * row_bytes);
        int4 *d = (int4 *)(rows + dst * row_bytes);
        for (int64_t k = 0; k < row_bytes / 16; ++k) d[k] = __ldg(s + k);
    } else {
        const int64_t *s = (const int64_t *)(rows + srcr * row_bytes);
        int64_t *d = (int64_t *)(rows + dst * row_bytes);
        for (int64_t k = 0; k < row_bytes / 8; ++k) d[k] = __ldg((const long long *)(s + k));
    }
}

// Pass C, per SLOT tile (2048 particles): survivors map to themselves, the
// tile's zero slots (ranks z0..z1-1) take the surplus children of the parents
// staged from the anchored slice of the surplus-parent list (merge walk), the
// full parent vector is written with one 32-byte store per thread, and every
// zero-slot row is overwritten by its parent's row in place (sources count >= 2
// and destinations count 0 are disjoint).
constexpr int CSTAGE = TILE + 2 * ANCHOR + 2;

// Shard geometry of pass C: this shard's zero slots have global zero ranks
// zoff + local rank; global surplus ranks [soff, soff + s_self) are this
// shard's own surplus children (local pairs, gathered by the next move); the
// rest arrive as rows in `recv`, ordered by global rank.
// Peer memory of the other shards (P2P over NVLink: CUDA-IPC mappings of their resample
// workspaces and state buffers).  The workspaces share one layout (same n), so one set of
// offsets locates a peer's surplus-parent list, surplus starts and rank anchors.
constexpr int SMC_MAX_SHARDS = 16;
struct PeerTab {
    const char *ws[SMC_MAX_SHARDS];    // each rank's resample workspace
    const char *rows[SMC_MAX_SHARDS];  // each rank's current state buffer
    int64_t off_sp_idx, off_sp_start, off_anchor;
};

struct ShardC {
    int64_t zoff, soff, s_self;  // s_self < 0: single GPU (all pairs local)
    const char *recv;
    char *rows;
    int64_t row_bytes;
    // P2P exchange (zsp_all != null): the offsets above come from the allgathered per-rank
    // (Z, S, P, active) on the device, and a surplus child on another rank is read from that
    // rank's memory directly -- no host plan, no host sync, no packed send / receive
    const uint32_t *zsp_all;
    int G, rank;
    PeerTab peers;
    int32_t *status;
};

// The surplus parent owning local surplus rank r of a shard: its rank anchors where they
// exist, a walk of at most ANCHOR starts from there; beyond them, binary search.
SMC_DEV int64_t surplus_owner(const int32_t *anchor, const int32_t *sp_start, int64_t n, int64_t P, int64_t r)
{
    int64_t p;
    if (r / ANCHOR < n / ANCHOR + 2) {
        p = __ldcg(&anchor[r / ANCHOR]);
        while (p + 1 < P && (int64_t)__ldcg(&sp_start[p + 1]) <= r) ++p;
    } else {
        int64_t lo = 0, hi = P;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)__ldcg(&sp_start[mid]) <= r) lo = mid; else hi = mid;
        }
        p = lo;
    }
    return p;
}

// COPY32 (one GPU, 32-byte rows): the value collection's in-place copy fused in -- every zero
// slot's row is overwritten by its parent's as soon as the parent is known (sources have
// count >= 2, destinations count 0: disjoint), saving the separate copy pass and
// its re-read of the parent vector.
// Pass C (the index-only variant) at 8 blocks per SM: 32 registers, and the partial-tile store
// staging aliased onto the parent staging (25.9 KB of shared memory instead of 35.4) -- a
// latency-bound pass, so the extra resident warps pay: the PF resample phase at 2^24 0.2025 -> 0.1956 ms
// (same-box A/B, profiles/r2_assign_occupancy_ab.txt)
#ifndef RS_ASSIGN_ALIAS
#define RS_ASSIGN_ALIAS 1
#endif
#ifndef RS_ASSIGN_MINB
#define RS_ASSIGN_MINB 8
#endif
template <bool SHARD, bool COPY32 = false>
__global__ void __launch_bounds__(RT, (!SHARD && !COPY32) ? RS_ASSIGN_MINB : 0) k_rs_assign(const int32_t *__restrict__ cin, int64_t n,
                                                  int32_t *__restrict__ parents, ShardC sc, Layout L)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    const int64_t t = blockIdx.x;
    // every load that does not depend on another issued together, before the first branch: the
    // block's chain of dependent round trips (header / zero ranks -> anchors -> staged slice) is
    // its whole cost (a latency-bound pass), so the first trip carries all of them
    const int32_t active = h->active, trivial = h->trivial;
    const int64_t z0 = __ldcg(&L.tile_z0[t]), z1 = __ldcg(&L.tile_z0[t + 1]);  // local zero ranks
    const int64_t Zl = h->Z_total, Sl = h->S_total, P = h->P_total;
    const uint32_t zword = __ldcg(&L.zmask[t * (TILE / 32) + (threadIdx.x >> 2)]);
    if (!active) return;
    if (trivial) {
        if (blockIdx.x == 0 && threadIdx.x == 0) parents[0] = 0;
        return;
    }
    __shared__ int32_t s_start[CSTAGE], s_idx[CSTAGE];
    // index-only variant: the partial-tile store staging reuses the parent staging (dead by then:
    // barrier below).  Not with the fused row copy, whose stores would wait on that barrier.
    constexpr bool kAlias = RS_ASSIGN_ALIAS && !SHARD && !COPY32;
    static_assert(tile_smem_elems<int32_t, RT, RI>() <= CSTAGE, "s_io fits in s_start");
    __shared__ int32_t s_io_own[kAlias ? 1 : tile_smem_elems<int32_t, RT, RI>()];
    int32_t *const s_io = kAlias ? s_start : s_io_own;
    __shared__ uint32_t sm32[RT / 32 + 1];
    __shared__ int64_t s_soffs[SMC_MAX_SHARDS + 1], s_zs[3];
    const int64_t tbase = t * TILE;
    const int64_t base = tbase + (int64_t)threadIdx.x * RI;
    if (SHARD && sc.zsp_all) {  // this rank's zero / surplus offsets from the allgathered counts
        if (threadIdx.x == 0) {
            int64_t zo = 0, so = 0;
            for (int r = 0; r < sc.G; ++r) {
                const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(sc.zsp_all) + r);
                s_soffs[r] = so;
                if (r == sc.rank) { s_zs[0] = zo; s_zs[1] = so; s_zs[2] = v.y; }
                zo += v.x;
                so += v.y;
            }
            s_soffs[sc.G] = so;
            // sum(counts) != N over all ranks: zero slots and surplus children do not pair up
            if (blockIdx.x == 0 && zo != so) raise_status(sc.status, SMC_ECOUNTS);
        }
        __syncthreads();
        sc.zoff = s_zs[0];
        sc.soff = s_zs[1];
        sc.s_self = s_zs[2];
    }
    const int64_t s_self = sc.s_self < 0 ? Sl : sc.s_self;
    const int64_t soff = sc.soff, zoff = sc.zoff;
    // length of this shard's local piece [soff, soff+s_self) ∩ [zoff, zoff+Zl) in global ranks
    const int64_t piece = max((int64_t)0, min(zoff + Zl, soff + s_self) - max(zoff, soff));
    // this thread's RI slots: one byte of the tile's zero-slot bitmask (pass B1); padding bits are 0
    (void)cin;
    const uint32_t zb = (zword >> (8 * (threadIdx.x & 3))) & 0xFFu;
    auto zero = [&](int j) { return ((zb >> j) & 1u) != 0; };
    const uint32_t nz = __popc(zb);
    // local surplus ranks this tile needs: [lo_s, hi_s)
    const int64_t lo_s = max(zoff + z0, soff) - soff, hi_s = min(zoff + z1, soff + s_self) - soff;
    uint32_t cnt = 0;
    if (hi_s > lo_s) {
        // surplus parents covering [lo_s, hi_s): from the rank anchors where they exist
        // (k_rs_ranks writes them for ranks < (n/ANCHOR + 2) ANCHOR), else by binary search --
        // a shard's pairs can sit at local surplus ranks beyond its n slots
        const int64_t acap = n / ANCHOR + 2;
        auto owner = [&](int64_t r) {  // last p with sp_start[p] <= r
            int64_t a = 0, b = P;
            while (b - a > 1) {
                const int64_t mid = (a + b) >> 1;
                if ((int64_t)__ldcg(&L.sp_start[mid]) <= r) a = mid; else b = mid;
            }
            return (uint32_t)a;
        };
        const uint32_t a0 = lo_s / ANCHOR < acap ? (uint32_t)__ldcg(&L.anchor[lo_s / ANCHOR]) : owner(lo_s);
        const int64_t ka = (hi_s - 1) / ANCHOR + 1;
        const uint32_t a1 = ka * ANCHOR >= Sl ? (uint32_t)(P - 1)
                          : ka < acap        ? (uint32_t)__ldcg(&L.anchor[ka])
                                             : owner(hi_s - 1);
        cnt = a1 - a0 + 1;
        for (uint32_t k = threadIdx.x; k < cnt; k += RT) {
            SMC_CHECK(k + 1 < (uint32_t)CSTAGE && a0 + k <= (uint64_t)n);
            s_start[k] = __ldcg(&L.sp_start[a0 + k]);
            s_idx[k] = __ldcg(&L.sp_idx[a0 + k]);
        }
    }
    if (threadIdx.x == 0) s_start[cnt] = 0x7fffffff;  // walk sentinel (cnt < CSTAGE)
    uint32_t tot;
    const uint32_t ex = block_exclusive_sum<RT, uint32_t>(nz, sm32, &tot);
    int32_t par[RI];
    uint32_t lo = 0;
    if (!SHARD) {
        // one GPU: zero ranks and surplus ranks are the same 32-bit numbers.  Each staged
        // surplus parent k writes itself into the tile's rank table for the ranks it covers,
        // [start_k, start_{k+1}) within [z0, z1); each zero slot then reads its parent by rank.
        __shared__ int32_t s_par[TILE];
        __shared__ uint32_t s_long[TILE / 32 + 1], s_nlong;  // runs longer than 32 ranks: block-wide
        const uint32_t zlo = (uint32_t)z0, zhi = (uint32_t)z1;
        if (threadIdx.x == 0) s_nlong = 0;
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt; k += RT) {
            const uint32_t r0 = max((uint32_t)s_start[k], zlo), r1 = min((uint32_t)s_start[k + 1], zhi);
            if (r1 > r0 + 32) {
                SMC_CHECK(s_nlong < TILE / 32 + 1);
                s_long[atomicAdd(&s_nlong, 1u)] = k;  // at most TILE / 32 such runs in a tile
                continue;
            }
            const int32_t pk = s_idx[k];
            SMC_CHECK(r1 <= r0 || (r1 <= zlo + TILE && pk >= 0 && pk < n));
            for (uint32_t r = r0; r < r1; ++r) s_par[r - zlo] = pk;
        }
        __syncthreads();
        for (uint32_t l = 0; l < s_nlong; ++l) {  // e.g. one parent with thousands of children
            const uint32_t k = s_long[l];
            const uint32_t r0 = max((uint32_t)s_start[k], zlo), r1 = min((uint32_t)s_start[k + 1], zhi);
            const int32_t pk = s_idx[k];
            SMC_CHECK(r1 <= zlo + TILE && pk >= 0 && pk < n);
            for (uint32_t r = r0 + threadIdx.x; r < r1; r += RT) s_par[r - zlo] = pk;
        }
        __syncthreads();
        uint32_t g = ex;  // tile-local zero rank of this thread's next zero slot
        const int32_t b32 = (int32_t)base;
#pragma unroll
        for (int j = 0; j < RI; ++j) {
            par[j] = b32 + j;  // survivors keep their slot
            SMC_CHECK(!zero(j) || g < (uint32_t)TILE);
            if (zero(j)) par[j] = s_par[g++];
        }
        if (COPY32) {  // 4 row loads in flight per thread, then their stores
            double *rows = (double *)sc.rows;
#pragma unroll
            for (int j0 = 0; j0 < RI; j0 += 4) {
                double4 v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (zero(j0 + j)) ld256(rows + (int64_t)par[j0 + j] * 4, v[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (zero(j0 + j)) st256(rows + (base + j0 + j) * 4, v[j]);
            }
        }
    } else {
        const int64_t zr = z0 + ex;  // first local zero rank
        int64_t g = zoff + zr;       // global zero rank of this thread's next zero slot
        if (nz && cnt) {
            const int64_t s0 = max(g, soff) - soff;
            uint32_t hi = cnt;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((int64_t)s_start[mid] <= s0) lo = mid; else hi = mid;
            }
        }
#pragma unroll
        for (int j = 0; j < RI; ++j) {
            par[j] = (int32_t)(base + j);
            if (zero(j)) {
                if (g >= soff && g < soff + s_self) {
                    const int64_t s = g - soff;
                    while (lo + 1 < cnt && (int64_t)s_start[lo + 1] <= s) ++lo;
                    SMC_CHECK(lo < cnt);
                    par[j] = s_idx[lo];
                } else if (sc.zsp_all) {  // surplus child on another shard: read from its memory (P2P)
                    int h = 0;
                    while (h + 1 < sc.G && s_soffs[h + 1] <= g) ++h;
                    const int64_t r = g - s_soffs[h];  // rank h's local surplus rank
                    const char *wh = sc.peers.ws[h];
                    const uint4 zh = __ldcg(reinterpret_cast<const uint4 *>(sc.zsp_all) + h);
                    const int64_t p = surplus_owner(reinterpret_cast<const int32_t *>(wh + sc.peers.off_anchor),
                                                    reinterpret_cast<const int32_t *>(wh + sc.peers.off_sp_start), n,
                                                    zh.z, r);
                    const int64_t src = __ldcg(reinterpret_cast<const int32_t *>(wh + sc.peers.off_sp_idx) + p);
                    const char *srow = sc.peers.rows[h] + src * sc.row_bytes;
                    char *dst = sc.rows + (base + j) * sc.row_bytes;
                    for (int64_t b = 0; b < sc.row_bytes; b += 8)
                        *(int64_t *)(dst + b) = __ldcg((const long long *)(srow + b));
                } else if (sc.recv) {  // surplus child on another shard: its row arrived in recv
                    const int64_t k = g < soff ? g - zoff : g - zoff - piece;
                    const char *src = sc.recv + k * sc.row_bytes;
                    char *dst = sc.rows + (base + j) * sc.row_bytes;
                    for (int64_t b = 0; b < sc.row_bytes; b += 8)
                        *(int64_t *)(dst + b) = __ldcg((const long long *)(src + b));
                }
                ++g;
            }
        }
    }
    if (kAlias) __syncthreads();  // every thread is done with s_start before the staging reuses it
    store_blocked<RT, RI, int32_t>(parents, tbase, n, par, s_io);  // coalesced
}

// Sender side of the cross-shard exchange: rows of this shard's surplus children
// with local surplus ranks [lo_r, lo_r + cnt_r), destination ranges back to back.
struct PackRanges {
    int64_t lo[64], cnt[64], off[64];
    int K;
    int64_t total;
};

__global__ void k_rs_pack(const char *__restrict__ rows, int64_t row_bytes, int64_t n, PackRanges pr,
                          char *__restrict__ out, Layout L)
{
    SMC_PDL_WAIT();
    const int64_t Sl = L.hdr->S_total, P = L.hdr->P_total;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < pr.total; k += (int64_t)gridDim.x * blockDim.x) {
        int r = 0;
        while (r + 1 < pr.K && k >= pr.off[r + 1]) ++r;
        const int64_t s = pr.lo[r] + (k - pr.off[r]);  // local surplus rank
        if (s >= Sl) continue;
        int64_t p;
        if (s / ANCHOR < n / ANCHOR + 2) {  // anchored ranks (k_rs_ranks)
            p = __ldcg(&L.anchor[s / ANCHOR]);
            while (p + 1 < P && (int64_t)__ldcg(&L.sp_start[p + 1]) <= s) ++p;  // <= ANCHOR steps
        } else {  // beyond the anchors: last p with sp_start[p] <= s
            int64_t lo = 0, hi = P;
            while (hi - lo > 1) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)__ldcg(&L.sp_start[mid]) <= s) lo = mid; else hi = mid;
            }
            p = lo;
        }
        const int64_t src = __ldcg(&L.sp_idx[p]);
        for (int64_t b = 0; b < row_bytes; b += 8)
            *(int64_t *)(out + k * row_bytes + b) = __ldg((const long long *)(rows + src * row_bytes + b));
    }
}

// In-place copy of every zero-count row from its parent.
// Rows other than 32 bytes (32-byte rows are copied inside pass C).  Sources (count >= 2)
// and destinations (count 0) are disjoint, so no snapshot is needed.  One slot
// per thread keeps occupancy (and so the number of row loads in flight) at the maximum.
constexpr int CB = 512;
__global__ void __launch_bounds__(CB) k_rs_copy(const int32_t *__restrict__ parents, char *rows, int64_t row_bytes,
                                                int64_t n, Layout L)
{
    SMC_PDL_WAIT();
    if (!L.hdr->active || L.hdr->trivial) return;
    const int64_t j = (int64_t)blockIdx.x * CB + threadIdx.x;
    if (j >= n) return;
    const int32_t p = __ldg(parents + j);
    if (p != j) copy_row(rows, row_bytes, j, p);
}

__global__ void k_rs_export_zsp(Layout L, uint32_t *out)
{
    SMC_PDL_WAIT();
    const RsHeader *h = L.hdr;
    const bool on = h->active && !h->trivial;
    out[0] = on ? h->Z_total : 0;
    out[1] = on ? h->S_total : 0;
    out[2] = on ? h->P_total : 0;
    out[3] = h->active;
}

__global__ void k_rs_reset(Layout L)
{
    SMC_PDL_WAIT();
    RsHeader *h = L.hdr;
    h->active = 1;
    h->trivial = 0;
    h->Z_total = h->S_total = h->P_total = 0;
}

__global__ void __launch_bounds__(RT) k_copy_inplace(char *rows, int64_t row_bytes, const int32_t *__restrict__ parents,
                                                     int64_t n, const int32_t *gate)
{
    SMC_PDL_WAIT();
    if (gate && *gate == 0) return;
    for (int64_t j = (int64_t)blockIdx.x * RT + threadIdx.x; j < n; j += (int64_t)gridDim.x * RT) {
        const int32_t p = parents[j];
        if (p != j) copy_row(rows, row_bytes, j, p);
    }
}

__global__ void __launch_bounds__(RT) k_gather(char *__restrict__ dst, const char *__restrict__ src, int64_t row_bytes,
                                               const int32_t *__restrict__ parents, int64_t n)
{
    SMC_PDL_WAIT();
    const int64_t words = row_bytes / 8;
    const int64_t total = n * words;
    for (int64_t e = (int64_t)blockIdx.x * RT + threadIdx.x; e < total; e += (int64_t)gridDim.x * RT) {
        const int64_t j = e / words, k = e - j * words;
        ((int64_t *)dst)[e] = __ldg((const long long *)src + (int64_t)parents[j] * words + k);
    }
}

// The multinomial draws' two kernels (m: the largest draw count; blocks past the call's
// own count exit at once).
// add: residual -- the histogram buffer holds the floors f_i (pass A), the counts add onto them
inline void launch_mn2(cudaStream_t s, int64_t n, int64_t m, Key key, uint64_t stream, const double *u, Layout L,
                       int add)
{
    const size_t sm = mn2_scatter_smem(n);
    static size_t s_set = 0;  // opt in to > 48 KB of dynamic shared memory once (per size)
    if (sm > s_set) {
        cudaFuncSetAttribute(k_mn2_scatter<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(k_mn2_scatter<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        s_set = sm;
    }
    const int dpt = mn_dpt(mn_geom(n).nb);
    const int64_t mch = (int64_t)MT * dpt;
    if (dpt == 6)
        smc_launch(k_mn2_scatter<6>, (unsigned)((m + mch - 1) / mch), MT, sm, s, n, key, stream, u, L);
    else
        smc_launch(k_mn2_scatter<12>, (unsigned)((m + mch - 1) / mch), MT, sm, s, n, key, stream, u, L);
    const size_t sc = mn2_count_smem(n);
    static size_t c_set = 0;
    if (sc > c_set) {
        cudaFuncSetAttribute(k_mn2_count<1024, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc);
        cudaFuncSetAttribute(k_mn2_count<1024, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc);
        c_set = sc;
    }
    if (2 * (sc + 1024) <= 233472) {  // two blocks per SM (228 KB, 1 KB reserved per block)
        static size_t c2_set = 0;
        if (sc > c2_set) {
            cudaFuncSetAttribute(k_mn2_count<512, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc);
            cudaFuncSetAttribute(k_mn2_count<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc);
            c2_set = sc;
        }
        if (add) smc_launch(k_mn2_count<512, true>, (unsigned)mn_geom(n).nb, 512, sc, s, n, L);
        else smc_launch(k_mn2_count<512, false>, (unsigned)mn_geom(n).nb, 512, sc, s, n, L);
    } else {
        if (add) smc_launch(k_mn2_count<1024, true>, (unsigned)mn_geom(n).nb, 1024, sc, s, n, L);
        else smc_launch(k_mn2_count<1024, false>, (unsigned)mn_geom(n).nb, 1024, sc, s, n, L);
    }
}

inline int grid_cap(int64_t blocks);
inline void launch_mn(cudaStream_t s, int64_t n, int64_t m, Key key, uint64_t stream, const double *u, Layout L,
                      int add)
{
    if (mn2_fits(n)) {
        launch_mn2(s, n, m, key, stream, u, L, add);
        return;
    }
    const unsigned gm = grid_cap((m + RT - 1) / RT);
    smc_launch(k_mn1_count, gm, RT, 0, s, n, key, stream, u, L);
    smc_launch(k_mn1_scan, 1, SB, 0, s, mn1_bins(n), n, L);
    smc_launch(k_mn1_starts, (unsigned)((mn1_bins(n) + 1 + RT - 1) / RT), RT, 0, s, n, L);
    smc_launch(k_mn1_scatter, gm, RT, 0, s, n, key, stream, u, L);
    smc_launch(k_mn1_assign, gm, RT, 0, s, n, L);
}

inline int grid_cap(int64_t blocks)
{
    return (int)(blocks < 1 ? 1 : (blocks > 148 * 16 ? 148 * 16 : blocks));
}

}  // namespace

extern "C" size_t smc_resample_workspace_bytes(int64_t n)
{
    if (n < 1) n = 1;
    return layout(nullptr, n).bytes;
}

extern "C" int smc_resample(int scheme, const double *w, const double *lw_raw, const smc_wstate *st, int64_t n,
                            int64_t m_out, uint64_t seed, uint64_t stream_index, uint64_t *ctr, const double *u,
                            int64_t n_u, int32_t *counts, int32_t *parents, void *rows, int64_t row_bytes,
                            const int32_t *gate, int32_t *status, void *ws, size_t ws_bytes, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (scheme < 0 || scheme > 5 || n < 1 || n >= ((int64_t)1 << 31) - TILE || m_out < 1 ||
        m_out >= ((int64_t)1 << 31))
        return smc_set_error(SMC_EINVAL, "smc_resample: bad scheme/size (scheme=%d n=%lld m=%lld)", scheme,
                             (long long)n, (long long)m_out);
    if (!w && (!lw_raw || !st)) return smc_set_error(SMC_EINVAL, "smc_resample: need w or (lw_raw, state)");
    if (!u && !ctr) return smc_set_error(SMC_EINVAL, "smc_resample: need uniforms or a stream counter");
    if ((parents || rows) && m_out != n)
        return smc_set_error(SMC_EINVAL, "smc_resample: parent map / copy need m_out == n");
    if (rows && !parents) return smc_set_error(SMC_EINVAL, "smc_resample: the row copy needs a parents buffer");
    if (rows && (row_bytes < 8 || (row_bytes & 7)))
        return smc_set_error(SMC_EINVAL, "smc_resample: row_bytes must be a positive multiple of 8");
    if (rows && row_bytes == 32 && ((uintptr_t)rows & 31))
        return smc_set_error(SMC_EINVAL, "smc_resample: 32-byte rows must be 32-byte aligned");
    if (counts && ((uintptr_t)counts & 15))
        return smc_set_error(SMC_EINVAL, "smc_resample: counts must be 16-byte aligned");
    if (!ws || ws_bytes < smc_resample_workspace_bytes(n))
        return smc_set_error(SMC_EWORKSPACE, "smc_resample: workspace too small");
    const int64_t nt = (n + TILE - 1) / TILE;
    Layout L = layout(ws, n);
    int L2 = 0;
    while (((int64_t)1 << L2) < n) ++L2;
    const double rscale = ldexp(1.0, 63 - L2);
    const Key key{(uint32_t)seed, (uint32_t)(seed >> 32)};
    WSrc src{w, lw_raw, st, n};
    const double mo = (double)m_out;

    launch_tiles(scheme, (unsigned)nt, s, src, n, mo, rscale, u, n_u, gate, status, L);
    if (nt <= (int64_t)SB * 8 / 32 * 32) {  // one pass with the tile sums in registers (N <= 2^24)
        const bool res = scheme == SMC_RESIDUAL || scheme == SMC_RESIDUAL_STRATIFIED || scheme == SMC_RESIDUAL_SYSTEMATIC;
        if (res)
            smc_launch(k_rs_scan1<true>, 1, SB, 0, s, scheme, n, nt, (uint64_t)m_out, key, stream_index, ctr, u, n_u,
                       gate, status, L);
        else
            smc_launch(k_rs_scan1<false>, 1, SB, 0, s, scheme, n, nt, (uint64_t)m_out, key, stream_index, ctr, u, n_u,
                       gate, status, L);
    } else {
        smc_launch(k_rs_scan, 1, SB, 0, s, scheme, n, nt, (uint64_t)m_out, key, stream_index, ctr, u, n_u, gate, status,
                   L, nullptr, 1, 0, n);
    }
    if (scheme == SMC_MULTINOMIAL || scheme == SMC_RESIDUAL) {
        const unsigned gm = grid_cap((m_out + RT - 1) / RT);
        smc_launch(k_rs_prefix, (unsigned)nt, RT, 0, s, scheme, src, n, mo, rscale, L);
        launch_mn(s, n, m_out, key, stream_index, u, L, scheme == SMC_RESIDUAL);
        smc_launch(k_rs_multinomial, gm, RT, 0, s, n, key, stream_index, u, L);  // exits unless mn_direct
    }
    int32_t *cout = counts ? counts : L.cnt;
    launch_counts(scheme, (unsigned)nt, s, src, n, mo, rscale, key, stream_index, u, cout, parents != nullptr, L);
    if (parents) {
        smc_launch(k_rs_zsp_scan, 1, SB, 0, s, nt, 1, status, L);
        smc_launch(k_rs_ranks, (unsigned)nt, RT, 0, s, cout, n, status, 0, L);
        if (rows && row_bytes == 32) {  // the value collection's copy fused into pass C
            smc_launch(k_rs_assign<false, true>, (unsigned)nt, RT, 0, s, cout, n, parents,
                       ShardC{0, 0, -1, nullptr, (char *)rows, 32, nullptr, 0, 0, {}, nullptr}, L);
        } else {
            smc_launch(k_rs_assign<false>, (unsigned)nt, RT, 0, s, cout, n, parents, ShardC{0, 0, -1, nullptr, nullptr, 0, nullptr, 0, 0, {}, nullptr}, L);
            if (rows)  // other row sizes: one moved row per thread, full occupancy
                smc_launch(k_rs_copy, (unsigned)((n + CB - 1) / CB), CB, 0, s, parents, (char *)rows, row_bytes, n, L);
        }
    }
    return smc_check_launch("smc_resample");
}

extern "C" int smc_replication_to_parents(const int32_t *counts, int64_t n, int32_t *parents, int32_t *status, void *ws,
                                          size_t ws_bytes, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    if (n < 1 || n >= ((int64_t)1 << 31) - TILE || !counts || !parents)
        return smc_set_error(SMC_EINVAL, "smc_replication_to_parents: bad args");
    if (!ws || ws_bytes < smc_resample_workspace_bytes(n))
        return smc_set_error(SMC_EWORKSPACE, "smc_replication_to_parents: workspace too small");
    const int64_t nt = (n + TILE - 1) / TILE;
    Layout L = layout(ws, n);
    if ((uintptr_t)counts & 15) return smc_set_error(SMC_EINVAL, "smc_replication_to_parents: counts alignment");
    smc_launch(k_rs_reset, 1, 1, 0, s, L);
    smc_launch(k_rs_aggs, (unsigned)nt, RT, 0, s, counts, n, L);
    smc_launch(k_rs_zsp_scan, 1, SB, 0, s, nt, 1, status, L);
    smc_launch(k_rs_ranks, (unsigned)nt, RT, 0, s, counts, n, status, 1, L);
    smc_launch(k_rs_assign<false>, (unsigned)nt, RT, 0, s, counts, n, parents, ShardC{0, 0, -1, nullptr, nullptr, 0, nullptr, 0, 0, {}, nullptr}, L);
    return smc_check_launch("smc_replication_to_parents");
}

extern "C" int smc_copy_rows_inplace(void *rows, int64_t row_bytes, const int32_t *parents, int64_t n,
                                     const int32_t *gate, void *stream)
{
    if (!rows || !parents || n < 1 || row_bytes < 8 || (row_bytes & 7) ||
        (row_bytes == 32 && ((uintptr_t)rows & 31)))
        return smc_set_error(SMC_EINVAL, "smc_copy_rows_inplace: bad args");
    smc_launch(k_copy_inplace, grid_cap((n + RT - 1) / RT), RT, 0, (cudaStream_t)stream, (char *)rows, row_bytes, parents,
                                                                                 n, gate);
    return smc_check_launch("smc_copy_rows_inplace");
}

extern "C" int smc_gather_rows(void *dst, const void *src, int64_t row_bytes, const int32_t *parents, int64_t n,
                               void *stream)
{
    if (!dst || !src || dst == src || !parents || n < 1 || row_bytes < 8 || (row_bytes & 7))
        return smc_set_error(SMC_EINVAL, "smc_gather_rows: bad args");
    smc_launch(k_gather, grid_cap((n * (row_bytes / 8) + RT - 1) / RT), RT, 0, (cudaStream_t)stream, 
        (char *)dst, (const char *)src, row_bytes, parents, n);
    return smc_check_launch("smc_gather_rows");
}

int smc_pf_set_move_ws(int on);  // smc_pf.cu

extern "C" int smc_debug_set(int key, int value)
{
    if (key == SMC_DEBUG_MOVE_WS) return smc_pf_set_move_ws(value);
    if (key != SMC_DEBUG_FORCE_EXACT_F) return smc_set_error(SMC_EINVAL, "smc_debug_set: unknown key %d", key);
    cudaError_t e = cudaMemcpyToSymbol(g_force_exact, &value, sizeof(int));
    return e == cudaSuccess ? SMC_OK : smc_set_error(SMC_ECUDA, "smc_debug_set: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Sharded (multi-GPU) resampling: the same kernels with global offsets; the
// host allgathers two tiny vectors between the phases.
// ---------------------------------------------------------------------------
static int shard_common(int scheme, const double *w, const double *lw_raw, const smc_wstate *st, int64_t n,
                        int64_t n_total, int64_t m_total, void *ws, size_t ws_bytes, const char *who)
{
    if (scheme < 0 || scheme > 5 || n < 1 || n >= ((int64_t)1 << 31) - TILE || n_total < n ||
        n_total >= ((int64_t)1 << 31) || m_total != n_total)
        return smc_set_error(SMC_EINVAL, "%s: bad sizes", who);
    if (!w && (!lw_raw || !st)) return smc_set_error(SMC_EINVAL, "%s: need w or (lw_raw, state)", who);
    if (!ws || ws_bytes < smc_resample_workspace_bytes(n)) return smc_set_error(SMC_EWORKSPACE, "%s: workspace", who);
    return SMC_OK;
}

static double shard_rscale(int64_t n_total)
{
    int L2 = 0;
    while (((int64_t)1 << L2) < n_total) ++L2;
    return ldexp(1.0, 63 - L2);
}

extern "C" int smc_resample_shard_totals(int scheme, const double *w, const double *lw_raw, const smc_wstate *st,
                                         int64_t n, int64_t n_total, int64_t m_total, const double *u, int64_t n_u,
                                         const int32_t *gate, int32_t *status, void *ws, size_t ws_bytes,
                                         uint64_t *totals_out, void *stream)
{
    int rc = shard_common(scheme, w, lw_raw, st, n, n_total, m_total, ws, ws_bytes, "smc_resample_shard_totals");
    if (rc) return rc;
    if (!totals_out) return smc_set_error(SMC_EINVAL, "smc_resample_shard_totals: totals_out");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nt = (n + TILE - 1) / TILE;
    Layout L = layout(ws, n);
    WSrc src{w, lw_raw, st, n_total};  // equal weights are 1 / N_total
    launch_tiles(scheme, (unsigned)nt, s, src, n, (double)m_total, shard_rscale(n_total), u, n_u, gate,
                                           status, L);
    smc_launch(k_rs_local_totals, 1, SB, 0, s, nt, gate, L, totals_out);
    return smc_check_launch("smc_resample_shard_totals");
}

extern "C" int smc_resample_shard_counts(int scheme, const double *w, const double *lw_raw, const smc_wstate *st,
                                         int64_t n, int64_t n_total, int64_t m_total, int G, int rank,
                                         const uint64_t *totals_all, uint64_t seed, uint64_t stream_index,
                                         uint64_t *ctr, const double *u, int64_t n_u, int32_t *counts,
                                         const int32_t *gate, int32_t *status, void *ws, size_t ws_bytes,
                                         uint32_t *zsp_out, void *stream)
{
    int rc = shard_common(scheme, w, lw_raw, st, n, n_total, m_total, ws, ws_bytes, "smc_resample_shard_counts");
    if (rc) return rc;
    if (G < 1 || rank < 0 || rank >= G || !totals_all || !zsp_out || (!u && !ctr))
        return smc_set_error(SMC_EINVAL, "smc_resample_shard_counts: bad shard args");
    if (counts && ((uintptr_t)counts & 15)) return smc_set_error(SMC_EINVAL, "smc_resample_shard_counts: counts");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nt = (n + TILE - 1) / TILE;
    Layout L = layout(ws, n);
    WSrc src{w, lw_raw, st, n_total};
    const Key key{(uint32_t)seed, (uint32_t)(seed >> 32)};
    const double rscale = shard_rscale(n_total), mo = (double)m_total;
    smc_launch(k_rs_scan, 1, SB, 0, s, scheme, n, nt, (uint64_t)m_total, key, stream_index, ctr, u, n_u, gate, status, L,
                               totals_all, G, rank, n_total);
    if (scheme == SMC_MULTINOMIAL || scheme == SMC_RESIDUAL) {
        const unsigned gm = grid_cap((m_total + RT - 1) / RT);
        smc_launch(k_rs_prefix, (unsigned)nt, RT, 0, s, scheme, src, n, mo, rscale, L);
        launch_mn(s, n, m_total, key, stream_index, u, L, scheme == SMC_RESIDUAL);
        smc_launch(k_rs_multinomial, gm, RT, 0, s, n, key, stream_index, u, L);  // exits unless mn_direct
    }
    int32_t *cout = counts ? counts : L.cnt;
    launch_counts(scheme, (unsigned)nt, s, src, n, mo, rscale, key, stream_index, u, cout, 1, L);
    smc_launch(k_rs_zsp_scan, 1, SB, 0, s, nt, 0, status, L);
    smc_launch(k_rs_ranks, (unsigned)nt, RT, 0, s, cout, n, status, 0, L);
    smc_launch(k_rs_export_zsp, 1, 1, 0, s, L, zsp_out);
    return smc_check_launch("smc_resample_shard_counts");
}

extern "C" int smc_resample_shard_pack(const void *rows, int64_t row_bytes, int64_t n, const int64_t *ranges, int K,
                                       void *sendbuf, void *ws, size_t ws_bytes, void *stream)
{
    if (!rows || row_bytes < 8 || (row_bytes & 7) || K < 0 || K > 64 || (K && (!ranges || !sendbuf)) || !ws ||
        n < 1 || ws_bytes < smc_resample_workspace_bytes(n))
        return smc_set_error(SMC_EINVAL, "smc_resample_shard_pack: bad args");
    PackRanges pr{};
    pr.K = K;
    int64_t off = 0;
    for (int r = 0; r < K; ++r) {
        pr.lo[r] = ranges[2 * r];
        pr.cnt[r] = ranges[2 * r + 1];
        pr.off[r] = off;
        off += pr.cnt[r];
    }
    pr.total = off;
    if (!off) return SMC_OK;
    Layout L = layout(ws, n);
    const int bs = 256;
    smc_launch(k_rs_pack, grid_cap((off + bs - 1) / bs), bs, 0, (cudaStream_t)stream, (const char *)rows, row_bytes, n, pr,
                                                                              (char *)sendbuf, L);
    return smc_check_launch("smc_resample_shard_pack");
}

extern "C" int smc_resample_shard_assign(const int32_t *counts, int64_t n, int64_t zoff, int64_t soff, int64_t s_self,
                                         const void *recv, void *rows, int64_t row_bytes, int32_t *parents, void *ws,
                                         size_t ws_bytes, void *stream)
{
    if (n < 1 || !parents || !ws || ws_bytes < smc_resample_workspace_bytes(n) || zoff < 0 || soff < 0 ||
        (recv && (!rows || row_bytes < 8 || (row_bytes & 7))))
        return smc_set_error(SMC_EINVAL, "smc_resample_shard_assign: bad args");
    const int64_t nt = (n + TILE - 1) / TILE;
    Layout L = layout(ws, n);
    const int32_t *cin = counts ? counts : L.cnt;
    smc_launch(k_rs_assign<true>, (unsigned)nt, RT, 0, (cudaStream_t)stream, 
        cin, n, parents, ShardC{zoff, soff, s_self, (const char *)recv, (char *)rows, row_bytes, nullptr, 0, 0, {}, nullptr}, L);
    return smc_check_launch("smc_resample_shard_assign");
}

extern "C" int smc_resample_shard_assign_p2p(const uint32_t *zsp_all, int G, int rank, const void *const *peer_ws,
                                             const void *const *peer_rows, int64_t n, void *rows, int64_t row_bytes,
                                             int32_t *parents, int32_t *status, void *ws, size_t ws_bytes,
                                             void *stream)
{
    if (n < 1 || !parents || !ws || ws_bytes < smc_resample_workspace_bytes(n) || !zsp_all || G < 1 ||
        G > SMC_MAX_SHARDS || rank < 0 || rank >= G || !peer_ws || !peer_rows || !rows || row_bytes < 8 ||
        (row_bytes & 7))
        return smc_set_error(SMC_EINVAL, "smc_resample_shard_assign_p2p: bad args");
    for (int r = 0; r < G; ++r)
        if (!peer_ws[r] || !peer_rows[r]) return smc_set_error(SMC_EINVAL, "smc_resample_shard_assign_p2p: peer %d", r);
    const int64_t nt = (n + TILE - 1) / TILE;
    Layout L = layout(ws, n);
    ShardC sc{0, 0, 0, nullptr, (char *)rows, row_bytes, zsp_all, G, rank, {}, status};
    for (int r = 0; r < G; ++r) {
        sc.peers.ws[r] = (const char *)peer_ws[r];
        sc.peers.rows[r] = (const char *)peer_rows[r];
    }
    sc.peers.off_sp_idx = (const char *)L.sp_idx - (const char *)ws;
    sc.peers.off_sp_start = (const char *)L.sp_start - (const char *)ws;
    sc.peers.off_anchor = (const char *)L.anchor - (const char *)ws;
    smc_launch(k_rs_assign<true>, (unsigned)nt, RT, 0, (cudaStream_t)stream, nullptr, n, parents, sc, L);
    return smc_check_launch("smc_resample_shard_assign_p2p");
}
