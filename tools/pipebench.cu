// Pipe-throughput micro-benchmark on B200 (tools only): warp instructions per SM per
// clock for DFMA, DADD, IMAD.WIDE.U32, IMAD (lo), LOP3, FFMA -- 8 independent chains
// per thread, 2^20 threads, 1024 iterations.
#include <cstdio>
#include <cstdint>
template <int F>
__global__ void __launch_bounds__(256) k(double *out, uint32_t seed)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double d[8];
    uint32_t u[8], v[8];
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { d[j] = 1.0 + 1e-9 * (i + j); u[j] = seed + i * 8 + j; v[j] = u[j] * 3; f[j] = 1.0f + 1e-6f * j; }
#pragma unroll 1
    for (int it = 0; it < 1024; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (F == 0) d[j] = __fma_rn(d[j], 0.999999999, 1e-10);
            if (F == 1) d[j] = __dadd_rn(d[j], 1e-10);
            if (F == 2) { const uint64_t p = (uint64_t)u[j] * 0xD2511F53u; u[j] = (uint32_t)p ^ (uint32_t)(p >> 32); }
            if (F == 3) u[j] = u[j] * 0xD2511F53u + v[j];
            if (F == 4) u[j] = (u[j] ^ v[j]) ^ (u[j] >> 3);
            if (F == 5) f[j] = __fmaf_rn(f[j], 0.9999999f, 1e-7f);
            if (F == 6) { d[j] += (double)(long long)(u[j] + v[j]); u[j] += 3; }            // I2F.F64.S64
            if (F == 7) { d[j] += (double)(int)(u[j] + v[j]); u[j] += 3; }                  // I2F.F64.S32
            if (F == 8) { d[j] += (double)((unsigned long long)u[j] << 21 | v[j]); u[j] += 3; }  // I2F.F64.U64
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j] + u[j] + f[j];
    out[i] = s;
}
int main()
{
    const int n = 1 << 20;
    double *d;
    cudaMalloc(&d, n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char *names[] = {"DFMA", "DADD", "IMAD.WIDE+LOP3", "IMAD(lo)", "LOP3+SHF", "FFMA", "I2F.F64.S64+DADD",
                           "I2F.F64.S32+DADD", "I2F.F64.U64+DADD"};
    for (int f = 0; f < 9; ++f) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            switch (f) {
            case 0: k<0><<<n / 256, 256>>>(d, 7); break;
            case 1: k<1><<<n / 256, 256>>>(d, 7); break;
            case 2: k<2><<<n / 256, 256>>>(d, 7); break;
            case 3: k<3><<<n / 256, 256>>>(d, 7); break;
            case 4: k<4><<<n / 256, 256>>>(d, 7); break;
            case 5: k<5><<<n / 256, 256>>>(d, 7); break;
            case 6: k<6><<<n / 256, 256>>>(d, 7); break;
            case 7: k<7><<<n / 256, 256>>>(d, 7); break;
            case 8: k<8><<<n / 256, 256>>>(d, 7); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        const double ops = (double)n * 8 * 1024;  // per-thread ops of the chain body
        printf("%-16s %8.3f ms  %7.2f thread-ops per SM per clk (at %d MHz, %d SMs)\n", names[f], best,
               ops / (best * 1e-3) / sms / (clk * 1e3), clk / 1000, sms);
    }
    return 0;
}
