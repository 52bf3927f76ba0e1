// smc_abi_common.cu -- version and host-side error reporting of the C ABI.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "smc_common.cuh"

static thread_local char g_err[512] = "";

int smc_set_error(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int smc_check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return smc_set_error(SMC_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return SMC_OK;
}

extern "C" int smc_abi_version(void) { return SMC_ABI_VERSION; }

extern "C" int smc_last_error(char *buf, size_t len)
{
    if (!buf || !len) return SMC_EINVAL;
    strncpy(buf, g_err, len - 1);
    buf[len - 1] = 0;
    return SMC_OK;
}

extern "C" int smc_check_failures(uint64_t *fails, uint64_t *first_line, char *file, size_t file_len)
{
    if (!fails || !first_line) return smc_set_error(SMC_EINVAL, "smc_check_failures: null");
    *fails = 0;
    *first_line = 0;
    const char *f = "";
    for (smc_chk_reader r : smc_chk_readers()) r(fails, first_line, &f);
    if (file && file_len) {
        size_t k = 0;
        for (; f[k] && k + 1 < file_len; ++k) file[k] = f[k];
        file[k] = 0;
    }
#if SMC_CHECKED
    return 1;  // a checked build
#else
    return 0;
#endif
}

extern "C" int smc_launch_count(uint64_t *out)
{
    if (!out) return SMC_EINVAL;
    *out = smc_launch_counter().load(std::memory_order_relaxed);
    return SMC_OK;
}
