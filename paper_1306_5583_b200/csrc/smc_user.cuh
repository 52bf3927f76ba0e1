// smc_user.cuh -- the device-side plugin surface for user particle kernels
// compiled at run time (NVRTC, smc_user_compile).  The GPU analogue of the
// reference's per-particle kernel `kernel(iter, SingleParticleView) -> int`
// (MoveAdapter :944-982):
//
//     #include "smc_user.cuh"
//     __device__ int my_move(smc::Particle &p, unsigned long long iter, const double *params)
//     {
//         p.state(0) += p.normal(0.0, 0.1);      // own row
//         p.slot(0) = -0.5 * p.state(0) * p.state(0);   // own scratch slot (e.g. incw)
//         return 1;                              // acceptance count contribution
//     }
//     SMC_USER_MOVE(my_move)
//
// One thread per particle; the own-slot contract of SPEC.md:396/:437 holds by
// construction: a kernel sees only its particle's state row, RNG stream
// (counter kept in a register, written back once) and scratch slot.
// Acceptance counts are summed exactly (integer atomics), so results do not
// depend on the launch configuration.
//
//     __device__ void my_eval(const smc::Particle &p, unsigned long long iter, const double *params,
//                             double *out)          // out[0..dim)
//     SMC_USER_EVAL(my_eval)
//
// Evaluators (monitor / path integrand) are pure: no RNG (counters are not
// written back), no state writes.
#pragma once

#include "smc_rng_device.cuh"

namespace smc {

struct Particle {
    double *x;          // state matrix base
    int64_t id;         // particle index (local to the shard)
    int64_t n;          // particles in the matrix
    int dim;
    int col_major;      // 0: row-major N x dim; 1: column-major
    uint64_t stream;    // global stream index = stream_base + id
    uint64_t ctr;       // the stream's counter (rng.py:159)
    Key key;
    double *scratch;    // N x sdim, row-major
    int sdim;

    SMC_DEV double &state(int pos) const { return col_major ? x[(int64_t)pos * n + id] : x[id * dim + pos]; }
    SMC_DEV double &slot(int k) const { return scratch[id * sdim + k]; }
    // RngStream draws (rng.py:186-215): uniform01, normal = mean + sd z, gamma(shape, scale)
    SMC_DEV double u01()
    {
        const double u = u01_at(ctr, stream, key);
        ctr += 1;
        return u;
    }
    SMC_DEV double normal(double mean, double sd)
    {
        const double z = normal_at(ctr, stream, key);
        ctr += 2;
        return mean + sd * z;
    }
    SMC_DEV double gamma(double shape, double scale) { return scale * gamma_from(ctr, stream, key, shape); }
};

SMC_DEV void user_acc_add(int a, unsigned long long *acc)
{
    // exact integer sum: warp reduce then one atomic per warp (order-free)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0 && a != 0 && acc) atomicAdd(acc, (unsigned long long)(long long)a);
}

}  // namespace smc

#define SMC_USER_MOVE(FN)                                                                                    \
    extern "C" __global__ void smc_user_entry(unsigned long long iter, double *x, long long n, int dim,       \
                                              int col_major, unsigned long long sbase, unsigned int k0,       \
                                              unsigned int k1, unsigned long long *ctrs, double *scratch,     \
                                              int sdim, const double *params, unsigned long long *acc)        \
    {                                                                                                         \
        const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;                                \
        int a = 0;                                                                                            \
        if (i < n) {                                                                                          \
            smc::Particle p{x, i, n, dim, col_major, sbase + (unsigned long long)i, ctrs[i], smc::Key{k0, k1}, \
                            scratch, sdim};                                                                   \
            a = FN(p, iter, params);                                                                          \
            ctrs[i] = p.ctr;                                                                                  \
        }                                                                                                     \
        smc::user_acc_add(a, acc);                                                                            \
    }                                                                                                         \
    extern "C" __global__ void smc_user_kind_move() {}

#define SMC_USER_EVAL(FN)                                                                                    \
    extern "C" __global__ void smc_user_entry(unsigned long long iter, double *x, long long n, int dim,       \
                                              int col_major, const double *params, double *out, int m)        \
    {                                                                                                         \
        const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;                                \
        if (i < n) {                                                                                          \
            const smc::Particle p{x, i, n, dim, col_major, 0, 0, smc::Key{0, 0}, nullptr, 0};                 \
            FN(p, iter, params, out + i * (long long)m);                                                      \
        }                                                                                                     \
    }                                                                                                         \
    extern "C" __global__ void smc_user_kind_eval() {}
