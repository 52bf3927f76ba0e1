// Micro-benchmark of the GMM log-likelihood inner loop on B200 (tools only):
// exp variants x (per-point log | product-of-mixtures log) over N particles x nd points.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include "../paper_1306_5583_b200/csrc/smc_common.cuh"
using namespace smc;

struct T2 { double hi, lo; };
__device__ T2 g_tab128[128];
__device__ T2 g_tab16[16];

SMC_DEV double exp_tab(double x, const T2 *tab, int bits, int deg)
{
    const int NT = 1 << bits;
    const double inv = NT / 0.6931471805599453;
    const double SH = 0x1.8p52;
    // ln2/NT split: hi with trailing zeros
    const double l2hi = 0x1.62e42fefa3800p-1 / NT, l2lo = 0x1.ef35793c76730p-45 / NT;
    double kd = __fma_rn(x, inv, SH);
    const int k = __double2loint(kd);
    kd -= SH;
    double r = __fma_rn(-kd, l2hi, x);
    r = __fma_rn(-kd, l2lo, r);
    double p;
    if (deg == 5) {
        p = __fma_rn(r, 1.0 / 120, 1.0 / 24);
        p = __fma_rn(r, p, 1.0 / 6);
        p = __fma_rn(r, p, 0.5);
        p = __fma_rn(r * r, p, r);
    } else {
        p = __fma_rn(r, 1.0 / 5040, 1.0 / 720);
        p = __fma_rn(r, p, 1.0 / 120);
        p = __fma_rn(r, p, 1.0 / 24);
        p = __fma_rn(r, p, 1.0 / 6);
        p = __fma_rn(r, p, 0.5);
        p = __fma_rn(r * r, p, r);
    }
    const T2 t = tab[k & (NT - 1)];
    const double m = __fma_rn(t.hi, p, t.lo) + t.hi;
    const int e = k >> bits;
    if (e < -1020 || e > 1020) return exp(x);
    return __hiloint2double(__double2hiint(m) + (e << 20), __double2loint(m));
}

SMC_DEV double exp_poly(double x)
{
    const double inv = 1.0 / 0.6931471805599453;
    const double SH = 0x1.8p52;
    double kd = __fma_rn(x, inv, SH);
    const int k = __double2loint(kd);
    kd -= SH;
    double r = __fma_rn(-kd, 0x1.62e42fefa3800p-1, x);
    r = __fma_rn(-kd, 0x1.ef35793c76730p-45, r);
    double p = 1.0 / 6227020800.0;  // 1/13!
    p = __fma_rn(r, p, 1.0 / 479001600.0);
    p = __fma_rn(r, p, 1.0 / 39916800.0);
    p = __fma_rn(r, p, 1.0 / 3628800.0);
    p = __fma_rn(r, p, 1.0 / 362880.0);
    p = __fma_rn(r, p, 1.0 / 40320.0);
    p = __fma_rn(r, p, 1.0 / 5040.0);
    p = __fma_rn(r, p, 1.0 / 720.0);
    p = __fma_rn(r, p, 1.0 / 120.0);
    p = __fma_rn(r, p, 1.0 / 24.0);
    p = __fma_rn(r, p, 1.0 / 6.0);
    p = __fma_rn(r, p, 0.5);
    p = __fma_rn(r * r, p, r);
    const double m = 1.0 + p;
    if (k < -1020 || k > 1020) return exp(x);
    return __hiloint2double(__double2hiint(m) + (k << 20), __double2loint(m));
}

template <int E, int PROD>
__global__ void __launch_bounds__(128) k_llh(const double *__restrict__ prm, const double *__restrict__ data, int nd,
                                             double *__restrict__ out, int n)
{
    extern __shared__ double s[];
    double *s_y = s;
    T2 *s_tab = (T2 *)(s + 4096);
    for (int k = threadIdx.x; k < nd; k += blockDim.x) s_y[k] = data[k];
    if (E == 1) for (int k = threadIdx.x; k < 128; k += blockDim.x) s_tab[k] = g_tab128[k];
    if (E == 3) for (int k = threadIdx.x; k < 16; k += blockDim.x) s_tab[k] = g_tab16[k];
    __syncthreads();
    const int i = blockIdx.x * 128 + threadIdx.x;
    if (i >= n) return;
    double mu[4], lam[4], om[4], c[4], b[4];
    for (int j = 0; j < 4; ++j) {
        mu[j] = prm[i * 12 + j];
        lam[j] = prm[i * 12 + 4 + j];
        om[j] = prm[i * 12 + 8 + j];
        c[j] = 0.5 * log(lam[j]) + log(om[j]);
        b[j] = -0.5 * lam[j];
    }
    double ll = -0.5 * nd * 1.8378770664093455;
    double m = 1.0;
    int ex = 0;
    for (int k = 0; k < nd; ++k) {
        const double yk = s_y[k];
        double lli = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double rr = yk - mu[j];
            if (E == 0) lli += om[j] * exp(0.5 * log(lam[j]) - 0.5 * lam[j] * rr * rr);
            else {
                const double x = __fma_rn(b[j], rr * rr, c[j]);
                if (E == 1) lli += exp_tab(x, s_tab, 7, 5);
                if (E == 2) lli += exp_tab(x, g_tab128, 7, 5);
                if (E == 3) lli += exp_tab(x, s_tab, 4, 7);
                if (E == 4) lli += exp_poly(x);
            }
        }
        if (PROD) {
            m *= lli;
            const int hi = __double2hiint(m);
            const int e = ((hi >> 20) & 0x7ff);
            if (e == 0 || e == 0x7ff) { ll += log(m); m = 1.0; }
            else { ex += e - 1023; m = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, __double2loint(m)); }
        } else {
            ll += smc_fm::log(lli);
        }
    }
    if (PROD) ll += smc_fm::log(m) + ex * 0.6931471805599453;
    out[i] = ll;
}

int main()
{
    const int n = 1 << 20, nd = 1000;
    std::vector<double> prm(n * 12), data(nd);
    uint64_t s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (s >> 11) * 0x1p-53; };
    for (int k = 0; k < nd; ++k) data[k] = -3 + 3 * (int)(rnd() * 4) + (rnd() - 0.5) * 1.5;
    for (int i = 0; i < n; ++i) {
        double sum = 0;
        for (int j = 0; j < 4; ++j) {
            prm[i * 12 + j] = -6 + 14 * rnd();
            prm[i * 12 + 4 + j] = 0.1 + 3 * rnd();
            prm[i * 12 + 8 + j] = 0.05 + rnd();
            sum += prm[i * 12 + 8 + j];
        }
        for (int j = 0; j < 4; ++j) prm[i * 12 + 8 + j] /= sum;
    }
    T2 t128[128], t16[16];
    for (int j = 0; j < 128; ++j) { long double v = exp2l(j / 128.0L); t128[j].hi = (double)v; t128[j].lo = (double)(v - (long double)t128[j].hi); }
    for (int j = 0; j < 16; ++j) { long double v = exp2l(j / 16.0L); t16[j].hi = (double)v; t16[j].lo = (double)(v - (long double)t16[j].hi); }
    cudaMemcpyToSymbol(g_tab128, t128, sizeof t128);
    cudaMemcpyToSymbol(g_tab16, t16, sizeof t16);
    double *dp, *dd, *dout;
    cudaMalloc(&dp, n * 12 * 8);
    cudaMalloc(&dd, nd * 8);
    cudaMalloc(&dout, n * 8 * 10);
    cudaMemcpy(dp, prm.data(), n * 12 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dd, data.data(), nd * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t sm = 4096 * 8 + 128 * 16;
    const char *names[] = {"libdevice exp, log/pt", "libdevice exp, prod", "tab128 smem, prod", "tab128 global, prod",
                           "tab16 smem, prod", "poly13, prod", "tab128 smem, log/pt"};
    for (int v = 0; v < 7; ++v) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            double *o = dout + (size_t)v * n;
            switch (v) {
            case 0: k_llh<0, 0><<<n / 128, 128, sm>>>(dp, dd, nd, o, n); break;
            case 1: k_llh<0, 1><<<n / 128, 128, sm>>>(dp, dd, nd, o, n); break;
            case 2: k_llh<1, 1><<<n / 128, 128, sm>>>(dp, dd, nd, o, n); break;
            case 3: k_llh<2, 1><<<n / 128, 128, sm>>>(dp, dd, nd, o, n); break;
            case 4: k_llh<3, 1><<<n / 128, 128, sm>>>(dp, dd, nd, o, n); break;
            case 5: k_llh<4, 1><<<n / 128, 128, sm>>>(dp, dd, nd, o, n); break;
            case 6: k_llh<1, 0><<<n / 128, 128, sm>>>(dp, dd, nd, o, n); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        std::vector<double> o(n), r(n);
        cudaMemcpy(o.data(), dout + (size_t)v * n, n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(r.data(), dout, n * 8, cudaMemcpyDeviceToHost);
        double md = 0, mr = 0;
        for (int i = 0; i < n; ++i) {
            double d = fabs(o[i] - r[i]);
            if (d > md) md = d;
            if (d / fabs(r[i]) > mr) mr = d / fabs(r[i]);
        }
        printf("%-26s %8.3f ms  %6.3f ps/comp-eval  max|d|=%.3g rel=%.3g  (ll[0]=%.12g)\n", names[v], best,
               best * 1e9 / ((double)n * nd * 4), md, mr, o[0]);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
