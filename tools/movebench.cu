// Micro-benchmark of the PF move's per-particle parts on B200 (tools only):
// 2^24 particles, 4 per thread, launch bounds of k_pf_move (256 x 4 blocks/SM).
//   philox8 : the 8 Philox blocks (53-bit draws) of one particle-step
//   bm4     : the 4 Box-Muller transforms alone (draw integers from a cheap hash)
//   normals : normals_at<4> (both)
#include <cstdio>
#include <cstdint>
#include "../paper_1306_5583_b200/csrc/smc_common.cuh"
using namespace smc;
constexpr int PPT = 4;
template <int F>
__global__ void __launch_bounds__(256, 4) k(double *out, int64_t n, const KeySched key)
{
    const int64_t base = (int64_t)blockIdx.x * 256 * PPT + threadIdx.x;
    double acc = 0.0;
    uint64_t iacc = 0;
#pragma unroll 1
    for (int q = 0; q < PPT; ++q) {
        const int64_t i = base + q * 256;
        const uint64_t c = (uint64_t)q * 8;
        if (F == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) iacc ^= draw53(c + j, (uint64_t)i, key);
        } else if (F == 1) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t h = (uint64_t)(i * 0x9E3779B97F4A7C15ull + j * 0xBF58476D1CE4E5B9ull);
                acc += box_muller53(h >> 11, (h * 0x94D049BB133111EBull) >> 11);
            }
        } else {
            double z[4];
            normals_at(c, (uint64_t)i, key, z);
            acc += z[0] + z[1] + z[2] + z[3];
        }
    }
    out[base] = acc + (double)iacc;
}
int main()
{
    const int64_t n = 1 << 24;
    double *d;
    cudaMalloc(&d, n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[] = {"philox8 (8 blocks)", "bm4 (4 Box-Muller)", "normals_at<4>"};
    const KeySched key = make_key_sched(1306);
    const int nb = (int)(n / (256 * PPT));
    for (int f = 0; f < 3; ++f) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (f == 0) k<0><<<nb, 256>>>(d, n, key);
            if (f == 1) k<1><<<nb, 256>>>(d, n, key);
            if (f == 2) k<2><<<nb, 256>>>(d, n, key);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("%-22s %8.4f ms per 2^24 particles\n", names[f], best);
    }
    return 0;
}
int smc_set_error(int c, const char *, ...) { return c; }
int smc_check_launch(const char *) { return 0; }
