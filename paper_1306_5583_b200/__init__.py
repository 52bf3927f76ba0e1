"""B200-native (sm_100a) SMC hot path of vSMC / smckit (arXiv 1306.5583).

Host orchestration in Python mirrors the smckit surface (rng, weights,
resample, core, exec, example-pf); every per-particle and per-weight
operation runs as a hand-written CUDA kernel in libsmcb200.so behind the C
ABI of include/smc_abi.h.  There is no CPU fallback.
"""

from . import _abi

_abi.load()  # build (nvcc, sm_100a) if missing, then dlopen: fail loudly otherwise

from .core import (COL_MAJOR, ROW_MAJOR, MonitorRecord, NormalizingConstant, ParticleSystem,  # noqa: E402
                   PathAccumulator, Sampler, SingleParticleView, StateMatrix, nc_add_log_weight, sampler_new)
from .exec import (Backend, MonitorEval, ParticleKernelOp, PathEval, apply_monitor_eval, apply_move,  # noqa: E402
                   apply_path_eval, make_op_from_kernel)
from .resample import (ResampleScheme, replication_to_parents, resample, resample_multinomial,  # noqa: E402
                       resample_residual, resample_residual_stratified, resample_residual_systematic,
                       resample_stratified, resample_systematic)
from .rng import (RngStream, RngStreamSet, fill_std_gamma, fill_std_normal, fill_u01, philox_block,  # noqa: E402
                  sample_gamma, sample_normal, sample_uniform01, std_gamma, std_normal, u01)
from .weights import WeightSet  # noqa: E402
from . import gmm, pf, user  # noqa: E402

__version__ = "0.1.0"

__all__ = [
    "RngStreamSet", "RngStream", "WeightSet", "ResampleScheme", "resample", "resample_multinomial",
    "resample_stratified", "resample_systematic", "resample_residual", "resample_residual_stratified",
    "resample_residual_systematic", "replication_to_parents", "StateMatrix", "ParticleSystem",
    "SingleParticleView", "Sampler", "MonitorRecord", "PathAccumulator", "NormalizingConstant", "Backend",
    "ParticleKernelOp", "MonitorEval", "PathEval", "apply_move", "apply_monitor_eval", "apply_path_eval",
    "make_op_from_kernel", "pf", "gmm", "user", "ROW_MAJOR", "COL_MAJOR", "nc_add_log_weight", "sampler_new",
    "philox_block", "u01", "std_normal", "std_gamma", "fill_u01", "fill_std_normal", "fill_std_gamma",
    "sample_uniform01", "sample_normal", "sample_gamma",
]
