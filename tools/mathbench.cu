// Micro-benchmark of the per-particle math on B200: cost per evaluation of the
// libdevice fp64 functions and of one Philox4x32-10 block (tools only).
#include <cstdio>
#include <cstdint>
#include "../paper_1306_5583_b200/csrc/smc_common.cuh"
using namespace smc;
template <int F>
__global__ void k(double *out, int64_t n, Key key)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    double x = 0.5 + (double)(i & 1023) * 1e-4;
#pragma unroll 1
    for (int r = 0; r < 8; ++r) {
        if (F == 0) acc += log(x + acc * 1e-300);
        if (F == 1) acc += cos(x * 6.283185307179586 + acc * 1e-300);
        if (F == 2) acc += sqrt(x + acc * 1e-300);
        if (F == 3) acc += exp(-x + acc * 1e-300);
        if (F == 4) acc += (double)draw53((uint64_t)r + (uint64_t)(acc * 1e-300), (uint64_t)i, key);
        if (F == 5) acc += normal_at((uint64_t)r * 2 + (uint64_t)(acc * 1e-300), (uint64_t)i, key);
        if (F == 6) acc += x * 1.0000001 + acc * 1e-300;
        if (F == 7) acc += smc_fm::log(x + acc * 1e-300);
        if (F == 8) acc += smc_fm::cos_bm(x * 6.283185307179586 + acc * 1e-300);
        if (F == 10) acc += smc_fm::log_core(x + acc * 1e-300);
        if (F == 9) acc += cospi(2.0 * x + acc * 1e-300);
        if (F == 11) {
            const uint64_t c = (uint64_t)r * 2 + (uint64_t)(acc * 1e-300);
            const double u1 = u01_at(c, (uint64_t)i, key), u2 = u01_at(c + 1, (uint64_t)i, key);
            acc += sqrt(-2.0 * smc_fm::log_core(1.0 - u1)) * cos((2.0 * 3.141592653589793) * u2);
        }
        x += 1e-3;
    }
    out[i] = acc;
}
int main()
{
    const int64_t n = 1 << 24;
    double *d;
    cudaMalloc(&d, n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[] = {"log", "cos", "sqrt", "exp", "philox+u53", "normal(2 philox+log+sqrt+cos)", "baseline",
                           "smc_fm::log", "smc_fm::cos_bm", "cospi(2x)", "smc_fm::log_core",
                           "normal(log_core+libdevice cos)"};
    for (int f = 0; f < 12; ++f) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            Key key{1306, 0};
            switch (f) {
            case 0: k<0><<<n / 256, 256>>>(d, n, key); break;
            case 1: k<1><<<n / 256, 256>>>(d, n, key); break;
            case 2: k<2><<<n / 256, 256>>>(d, n, key); break;
            case 3: k<3><<<n / 256, 256>>>(d, n, key); break;
            case 4: k<4><<<n / 256, 256>>>(d, n, key); break;
            case 5: k<5><<<n / 256, 256>>>(d, n, key); break;
            case 6: k<6><<<n / 256, 256>>>(d, n, key); break;
            case 7: k<7><<<n / 256, 256>>>(d, n, key); break;
            case 8: k<8><<<n / 256, 256>>>(d, n, key); break;
            case 9: k<9><<<n / 256, 256>>>(d, n, key); break;
            case 10: k<10><<<n / 256, 256>>>(d, n, key); break;
            case 11: k<11><<<n / 256, 256>>>(d, n, key); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("%-34s %8.3f ms for %lld x 8 evals = %6.2f ps/eval\n", names[f], ms, (long long)n, ms * 1e9 / (n * 8.0));
        }
    }
    return 0;
}
int smc_set_error(int c, const char *, ...) { return c; }
int smc_check_launch(const char *) { return 0; }
