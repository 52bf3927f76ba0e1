// smc_user.cu -- run-time compiled user particle kernels (the generic
// `kernel(iter, SingleParticleView) -> int` plugin path of SPEC.md:384-387 /
// PAPER.md:866-982 on the GPU).
//
// smc_user_compile: NVRTC compiles the user's CUDA source (which includes
// smc_user.cuh and ends with SMC_USER_MOVE / SMC_USER_EVAL) to an sm_100a
// cubin; the driver loads it and resolves `smc_user_entry`.  libnvrtc and
// libcuda are dlopen'ed on first use, so the library itself links neither
// (it must load on the CPU-only build host).  Launches go through
// cuLaunchKernel on the caller's stream.
#include <dlfcn.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "smc_common.cuh"

namespace {

typedef int nvrtcResult_t;
typedef void *nvrtcProgram_t;
typedef int CUresult_t;
typedef void *CUmodule_t;
typedef void *CUfunction_t;

struct Api {
    bool ok = false;
    std::string why;
    nvrtcResult_t (*CreateProgram)(nvrtcProgram_t *, const char *, const char *, int, const char *const *,
                                   const char *const *);
    nvrtcResult_t (*CompileProgram)(nvrtcProgram_t, int, const char *const *);
    nvrtcResult_t (*GetProgramLogSize)(nvrtcProgram_t, size_t *);
    nvrtcResult_t (*GetProgramLog)(nvrtcProgram_t, char *);
    nvrtcResult_t (*GetCUBINSize)(nvrtcProgram_t, size_t *);
    nvrtcResult_t (*GetCUBIN)(nvrtcProgram_t, char *);
    nvrtcResult_t (*DestroyProgram)(nvrtcProgram_t *);
    const char *(*GetErrorString)(nvrtcResult_t);
    CUresult_t (*ModuleLoadData)(CUmodule_t *, const void *);
    CUresult_t (*ModuleGetFunction)(CUfunction_t *, CUmodule_t, const char *);
    CUresult_t (*ModuleUnload)(CUmodule_t);
    CUresult_t (*LaunchKernel)(CUfunction_t, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                               void *, void **, void **);
    CUresult_t (*CuGetErrorString)(CUresult_t, const char **);
};

Api g_api;
std::once_flag g_once;

void *open_first(const char *const *names)
{
    for (int i = 0; names[i]; ++i)
        if (void *h = dlopen(names[i], RTLD_NOW | RTLD_GLOBAL)) return h;
    return nullptr;
}

template <typename F>
bool sym(void *h, const char *name, F &f)
{
    f = reinterpret_cast<F>(dlsym(h, name));
    return f != nullptr;
}

void load_api()
{
    static const char *nvrtc_names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                                        nullptr};
    static const char *cuda_names[] = {"libcuda.so.1", "libcuda.so", nullptr};
    void *hn = open_first(nvrtc_names);
    if (!hn) { g_api.why = "libnvrtc not found"; return; }
    void *hc = open_first(cuda_names);
    if (!hc) { g_api.why = "libcuda (the driver) not found"; return; }
    bool ok = sym(hn, "nvrtcCreateProgram", g_api.CreateProgram) && sym(hn, "nvrtcCompileProgram", g_api.CompileProgram) &&
              sym(hn, "nvrtcGetProgramLogSize", g_api.GetProgramLogSize) &&
              sym(hn, "nvrtcGetProgramLog", g_api.GetProgramLog) && sym(hn, "nvrtcGetCUBINSize", g_api.GetCUBINSize) &&
              sym(hn, "nvrtcGetCUBIN", g_api.GetCUBIN) && sym(hn, "nvrtcDestroyProgram", g_api.DestroyProgram) &&
              sym(hn, "nvrtcGetErrorString", g_api.GetErrorString) &&
              sym(hc, "cuModuleLoadData", g_api.ModuleLoadData) &&
              sym(hc, "cuModuleGetFunction", g_api.ModuleGetFunction) && sym(hc, "cuModuleUnload", g_api.ModuleUnload) &&
              sym(hc, "cuLaunchKernel", g_api.LaunchKernel) && sym(hc, "cuGetErrorString", g_api.CuGetErrorString);
    if (!ok) { g_api.why = "missing NVRTC / driver symbols"; return; }
    g_api.ok = true;
}

struct UserModule {
    CUmodule_t mod = nullptr;
    CUfunction_t fn = nullptr;
    int kind = 0;  // SMC_USER_MOVE / SMC_USER_EVAL
};

int cu_err(CUresult_t r, const char *what)
{
    const char *s = "?";
    if (g_api.CuGetErrorString) g_api.CuGetErrorString(r, &s);
    return smc_set_error(SMC_ECUDA, "%s: CUDA driver error %d (%s)", what, r, s);
}

}  // namespace

extern "C" int smc_user_compile(const char *source, const char *const *options, int n_options, void **module_out,
                                char *log, size_t log_bytes)
{
    if (!source || !module_out || n_options < 0 || (n_options && !options))
        return smc_set_error(SMC_EINVAL, "smc_user_compile: bad args");
    *module_out = nullptr;
    if (log && log_bytes) log[0] = 0;
    std::call_once(g_once, load_api);
    if (!g_api.ok) return smc_set_error(SMC_ECUDA, "smc_user_compile: %s", g_api.why.c_str());
    cudaFree(nullptr);  // make the device's primary context current for the driver API
    nvrtcProgram_t prog = nullptr;
    nvrtcResult_t r = g_api.CreateProgram(&prog, source, "smc_user_kernel.cu", 0, nullptr, nullptr);
    if (r) return smc_set_error(SMC_EINVAL, "smc_user_compile: nvrtcCreateProgram: %s", g_api.GetErrorString(r));
    std::vector<const char *> opts = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17", "-lineinfo"};
    for (int i = 0; i < n_options; ++i) opts.push_back(options[i]);
    r = g_api.CompileProgram(prog, (int)opts.size(), opts.data());
    size_t ls = 0;
    g_api.GetProgramLogSize(prog, &ls);
    if (log && log_bytes && ls > 1) {
        std::vector<char> buf(ls + 1, 0);
        g_api.GetProgramLog(prog, buf.data());
        snprintf(log, log_bytes, "%s", buf.data());
    }
    if (r) {
        g_api.DestroyProgram(&prog);
        return smc_set_error(SMC_EINVAL, "smc_user_compile: compilation failed (%s); see the log",
                             g_api.GetErrorString(r));
    }
    size_t nb = 0;
    g_api.GetCUBINSize(prog, &nb);
    std::vector<char> cubin(nb);
    g_api.GetCUBIN(prog, cubin.data());
    g_api.DestroyProgram(&prog);
    UserModule *m = new UserModule;
    CUresult_t cr = g_api.ModuleLoadData(&m->mod, cubin.data());
    if (cr) { delete m; return cu_err(cr, "smc_user_compile: cuModuleLoadData"); }
    CUfunction_t probe = nullptr;
    if (g_api.ModuleGetFunction(&probe, m->mod, "smc_user_kind_move") == 0) m->kind = SMC_USER_MOVE;
    else if (g_api.ModuleGetFunction(&probe, m->mod, "smc_user_kind_eval") == 0) m->kind = SMC_USER_EVAL;
    cr = m->kind ? g_api.ModuleGetFunction(&m->fn, m->mod, "smc_user_entry") : 1;
    if (cr || !m->kind) {
        g_api.ModuleUnload(m->mod);
        delete m;
        return smc_set_error(SMC_EINVAL, "smc_user_compile: the source must end with SMC_USER_MOVE(fn) or "
                                         "SMC_USER_EVAL(fn) (smc_user.cuh)");
    }
    *module_out = m;
    return SMC_OK;
}

extern "C" int smc_user_kind(const void *module)
{
    return module ? static_cast<const UserModule *>(module)->kind : 0;
}

extern "C" int smc_user_free(void *module)
{
    if (!module) return SMC_OK;
    UserModule *m = static_cast<UserModule *>(module);
    if (g_api.ok && m->mod) g_api.ModuleUnload(m->mod);
    delete m;
    return SMC_OK;
}

extern "C" int smc_user_launch_move(void *module, uint64_t iter, double *x, int64_t n, int dim, int col_major,
                                    uint64_t stream_base, uint64_t seed, uint64_t *ctrs, double *scratch, int sdim,
                                    const double *params, unsigned long long *accepted, void *stream)
{
    UserModule *m = static_cast<UserModule *>(module);
    if (!m || m->kind != SMC_USER_MOVE) return smc_set_error(SMC_EINVAL, "smc_user_launch_move: not a move module");
    if (n < 1 || dim < 1 || !x || !ctrs || sdim < 0 || (sdim > 0 && !scratch))
        return smc_set_error(SMC_EINVAL, "smc_user_launch_move: bad args");
    unsigned long long it = iter, sb = stream_base;
    long long nn = n;
    unsigned k0 = (unsigned)seed, k1 = (unsigned)(seed >> 32);
    void *args[] = {&it, &x, &nn, &dim, &col_major, &sb, &k0, &k1, &ctrs, &scratch, &sdim, &params, &accepted};
    const unsigned nb = (unsigned)((n + 255) / 256);
    CUresult_t cr = g_api.LaunchKernel(m->fn, nb, 1, 1, 256, 1, 1, 0, stream, args, nullptr);
    if (cr) return cu_err(cr, "smc_user_launch_move");
    SMC_COUNT_LAUNCH();
    return smc_check_launch("smc_user_launch_move");
}

extern "C" int smc_user_launch_eval(void *module, uint64_t iter, const double *x, int64_t n, int dim, int col_major,
                                    const double *params, double *out, int m_dim, void *stream)
{
    UserModule *m = static_cast<UserModule *>(module);
    if (!m || m->kind != SMC_USER_EVAL) return smc_set_error(SMC_EINVAL, "smc_user_launch_eval: not an eval module");
    if (n < 1 || dim < 1 || !x || !out || m_dim < 1) return smc_set_error(SMC_EINVAL, "smc_user_launch_eval: bad args");
    unsigned long long it = iter;
    long long nn = n;
    void *args[] = {&it, &x, &nn, &dim, &col_major, &params, &out, &m_dim};
    const unsigned nb = (unsigned)((n + 255) / 256);
    CUresult_t cr = g_api.LaunchKernel(m->fn, nb, 1, 1, 256, 1, 1, 0, stream, args, nullptr);
    if (cr) return cu_err(cr, "smc_user_launch_eval");
    SMC_COUNT_LAUNCH();
    return smc_check_launch("smc_user_launch_eval");
}
