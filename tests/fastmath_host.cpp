// Host build of paper_1306_5583_b200/csrc/smc_fastmath.h for the accuracy test.
#include "../paper_1306_5583_b200/csrc/smc_fastmath.h"
extern "C" void fm_log(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::log(x[i]); }
extern "C" void fm_cos(const double *x, double *y, long n) { for (long i = 0; i < n; ++i) y[i] = smc_fm::cos(x[i]); }
