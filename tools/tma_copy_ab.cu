// A/B of the resample's particle copy (north_star item 4: "the particle copy
// as a TMA/shared-memory-staged gather"): the in-place copy of 32-byte state rows (PF: N x 4
// f64) from their parents, as
//   (a) one 256-bit LDG + one 256-bit STG per moved row (what k_rs_assign<copy> does), and
//   (b) TMA: per warp, the elected lane gathers 4 parent rows into shared memory with
//       cp.async.bulk.tensor.2d.tile::gather4 (mbarrier completion) and scatters them to their
//       4 destination rows with tile::scatter4 -- no per-row thread instructions, 8 groups of
//       4 rows in flight per warp.
// Same synthetic map for both: destinations = the zero-count slots (a fraction f of all
// rows), sources = surplus parents (disjoint from destinations).  Timed with CUDA
// events; bytes = 64 per moved row (32 read + 32 written).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_copy_ab tools/tma_copy_ab.cu -lcuda
//   tools/tma_copy_ab [log2N=24] [moved fraction=0.55]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } \
    } while (0)

__global__ void k_copy_ldst(double *x, const int32_t *dst, const int32_t *src, int64_t m)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        double a, b, c, d;
        const double *p = x + 4 * (int64_t)__ldg(src + k);
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
        double *q = x + 4 * (int64_t)__ldg(dst + k);
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(q), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
    }
}

constexpr int STAGES = 8;  // groups of 4 rows in flight per warp

__global__ void __launch_bounds__(256) k_copy_tma(const __grid_constant__ CUtensorMap tmap, const int32_t *dst,
                                                  const int32_t *src, int64_t m)
{
    __shared__ __align__(128) double buf[8][STAGES][16];  // per warp: STAGES x (4 rows x 4 f64)
    __shared__ __align__(8) uint64_t bar[8][STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t tm = reinterpret_cast<uint64_t>(&tmap);
    if (lane == 0)
        for (int s = 0; s < STAGES; ++s) {
            const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t groups = (m + 3) / 4;
    const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
    uint32_t phase[STAGES] = {0};
    if (lane != 0) return;
    for (int64_t g0 = gw; g0 < groups; g0 += nw * STAGES) {
        int n_in = 0;
        for (int s = 0; s < STAGES; ++s) {  // issue up to STAGES gathers
            const int64_t g = g0 + (int64_t)s * nw;
            if (g >= groups) break;
            int r[4];
            for (int j = 0; j < 4; ++j) {
                const int64_t k = min(g * 4 + j, m - 1);  // a short last group repeats its last row
                r[j] = __ldg(src + k);
            }
            const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(&buf[warp][s][0]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 128;" ::"r"(b) : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
                "l"(tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(b)
                : "memory");
            ++n_in;
        }
        for (int s = 0; s < n_in; ++s) {  // as each lands, scatter it to its destinations
            const int64_t g = g0 + (int64_t)s * nw;
            const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(b), "r"(phase[s])
                    : "memory");
            phase[s] ^= 1;
            int r[4];
            for (int j = 0; j < 4; ++j) {
                const int64_t k = min(g * 4 + j, m - 1);
                r[j] = __ldg(dst + k);
            }
            const uint32_t sp = (uint32_t)__cvta_generic_to_shared(&buf[warp][s][0]);
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                         ::"l"(tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sp)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging reusable
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv)
{
    const int lg = argc > 1 ? atoi(argv[1]) : 24;
    const double f = argc > 2 ? atof(argv[2]) : 0.55;
    const int64_t n = (int64_t)1 << lg;
    // synthetic parent map: every slot is a destination with probability f (its parent a random
    // non-destination): the PF's zero-count slots and surplus parents
    std::mt19937_64 rng(1306);
    std::vector<char> isdst(n);
    std::vector<int32_t> srcs;
    for (int64_t i = 0; i < n; ++i) {
        isdst[i] = std::uniform_real_distribution<double>(0, 1)(rng) < f;
        if (!isdst[i]) srcs.push_back((int32_t)i);
    }
    std::vector<int32_t> dst, src;
    for (int64_t i = 0; i < n; ++i)
        if (isdst[i]) {
            dst.push_back((int32_t)i);
            src.push_back(srcs[std::uniform_int_distribution<size_t>(0, srcs.size() - 1)(rng)]);
        }
    const int64_t m = (int64_t)dst.size();
    double *x, *x2;
    int32_t *d_dst, *d_src;
    CK(cudaMalloc(&x, n * 32));
    CK(cudaMalloc(&x2, n * 32));
    CK(cudaMalloc(&d_dst, m * 4));
    CK(cudaMalloc(&d_src, m * 4));
    CK(cudaMemcpy(d_dst, dst.data(), m * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_src, src.data(), m * 4, cudaMemcpyHostToDevice));
    std::vector<double> h(n * 4);
    for (int64_t i = 0; i < n * 4; ++i) h[i] = (double)i;
    CK(cudaMemcpy(x, h.data(), n * 32, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x2, h.data(), n * 32, cudaMemcpyHostToDevice));

    CUtensorMap tmap;
    cuuint64_t gdim[2] = {4, (cuuint64_t)n}, gstride[1] = {32};
    cuuint32_t box[2] = {4, 1}, estr[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x2, gdim, gstride, box, estr,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed: %d\n", (int)cr); return 1; }

    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int reps = 20;
    auto time = [&](auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms / reps;
    };
    int dev;
    cudaGetDevice(&dev);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const float ta = time([&] { k_copy_ldst<<<sms * 16, 256>>>(x, d_dst, d_src, m); });
    const float tb = time([&] { k_copy_tma<<<sms * 8, 256>>>(tmap, d_dst, d_src, m); });
    CK(cudaGetLastError());
    std::vector<double> ha(n * 4), hb(n * 4);
    CK(cudaMemcpy(ha.data(), x, n * 32, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hb.data(), x2, n * 32, cudaMemcpyDeviceToHost));
    bool same = ha == hb;
    const double bytes = 64.0 * m;
    printf("{\"n\": %lld, \"moved\": %lld, \"moved_frac\": %.4f, \"ldst_ms\": %.4f, \"ldst_GBps\": %.1f, "
           "\"tma_ms\": %.4f, \"tma_GBps\": %.1f, \"same_result\": %s}\n",
           (long long)n, (long long)m, (double)m / n, ta, bytes / ta / 1e6, tb, bytes / tb / 1e6, same ? "true" : "false");
    return same ? 0 : 2;
}
