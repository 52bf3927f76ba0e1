// Host build of paper_1306_5583_b200/csrc/smc_fastmath.h for the accuracy test.
#include "../paper_1306_5583_b200/csrc/smc_fastmath.h"
extern "C" void fm_log(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::log(x[i]); }
extern "C" void fm_cos_bm(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::cos_bm(x[i]); }
extern "C" void fm_sqrt_bm(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::sqrt_bm(x[i]); }
extern "C" void fm_exp(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::exp(x[i], smc_fm::kExpTab); }
extern "C" double fm_logprod(const double *x, long n)
{
    smc_fm::LogProd lp;
    for (long i = 0; i < n; ++i) lp.add(x[i]);
    return lp.result();
}
extern "C" void fm_exp_weight(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::exp_weight(x[i]); }
extern "C" void fm_exp_nonpos(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::exp_nonpos(x[i], smc_fm::kExpTab); }
extern "C" void fm_div10(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::div10(x[i]); }
extern "C" void fm_exp_nonpos256(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::exp_nonpos256(x[i], smc_fm::kExpTab256); }
extern "C" void fm_exp_nonpos_cb(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::exp_nonpos_cb(x[i], smc_fm::kExpTab); }
