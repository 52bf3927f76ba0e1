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

extern "C" int smc_launch_count(uint64_t *out)
{
    if (!out) return SMC_EINVAL;
    *out = smc_launch_counter().load(std::memory_order_relaxed);
    return SMC_OK;
}
