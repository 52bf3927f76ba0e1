"""Benchmark: PF particle-steps/s at N = 2^24 on B200 (BASELINE.json metric, config 2).

A "step" is one Sampler.iterate() of the paper's particle filter: cv_move +
add_log_weight (fused lse/ESS), the ESS decision, systematic resampling with
the parent map and the in-place state copy, set_equal_weight and the "pos"
monitor -- the whole hot path, inputs resident in HBM (X is 512 MiB at 2^24,
larger than the 126 MB L2, so no flush is needed between steps).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle
(C restatement of the reference algorithm; OpenMP over all host cores for the
per-particle loops, sequential normalization/resampling as SPEC.md:99,:185 pin).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT = 1 << 24       # config 2: one B200
N_SHARDED = 1 << 28       # config 4: the whole filter sharded over G B200 (2^28 / G particles per GPU)
METRIC = "PF particle-steps/sec at N=2^24 (resample+copy GB/s vs HBM peak reported alongside)"
UNIT = "particle-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)  # ~0.55 s timed: several clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--particles", "--n", dest="n", type=int, default=None,
                    help="particles per GPU (default: 2^24 on one GPU -- config 2 -- and 2^28 / G on G > 1 "
                         "GPUs -- config 4, strong scaling); use --particles under torchrun: it claims --n*")
    ap.add_argument("--scheme", default="systematic")
    ap.add_argument("--config", type=int, choices=(2, 4), default=None,
                    help="2: N=2^24 per GPU (default on one GPU); 4: N=2^28 in total, sharded over the GPUs "
                         "(default on G > 1; --config 4 --gpus 1 runs the whole 2^28 filter on one GPU, the "
                         "same-config single-GPU point of the strong-scaling curve)")
    ap.add_argument("--no-schemes", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gmm", action="store_true")
    ap.add_argument("--no-config1", action="store_true")
    return ap.parse_args()


def workload(n, world, scheme, strong):
    """(scaling, config) of the JSON line: config 2 on one GPU, config 4 (2^28 in total) on G > 1.
    Both arms print exactly this config dict (the driver compares them)."""
    if strong:
        name = (f"PF config 4: N=2^{(n * world).bit_length() - 1} particles in total sharded over {world} GPUs "
                f"(2^{n.bit_length() - 1} per GPU), ")
    else:
        name = f"PF config 2: N=2^{n.bit_length() - 1} particles per GPU, "
    name += f"{scheme} resampling at ESS<N/2, 4-dim state, Student-t(10) likelihood, 100-obs model track"
    return ("strong" if strong else "weak"), {"workload": name, "n_particles": n * world, "scheme": scheme}


def config_of(args, world):
    return args.config if args.config is not None else (2 if world == 1 else 4)


def particles_per_gpu(args, world):
    if args.n is not None:
        return args.n
    return N_DEFAULT if config_of(args, world) == 2 else N_SHARDED // world


def is_strong(args, world):
    """Config 4 fixes the TOTAL work (2^28): strong scaling; config 2 / --particles fix it per GPU."""
    return args.n is None and config_of(args, world) == 4


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # one persistent nvidia-smi sampling every 100 ms (the profiling recipe's clocks line)
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        for line in self._p.stdout:
            if self._stop.is_set():
                break
            if line.strip():
                self.rows.append([c.strip() for c in line.split(",")])

    def __enter__(self):
        self._p = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.15)  # the first sample lands before the timed region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._p is not None:
            self._p.terminate()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        mx = max(float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 5 + k and r[5 + k] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------- CPU side ---
def cpu_baseline_pf(n, steps, scheme, obs, threads):
    """Oracle PF on the host cores: initialize untimed, then `steps` timed iterate()s."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O

    L = O.lib()

    class Sys(C.Structure):
        _fields_ = [("n", C.c_int64), ("x", C.c_void_p), ("lw", C.c_void_p), ("w", C.c_void_p),
                    ("incw", C.c_void_p), ("ctrs", C.c_void_p), ("counts", C.c_void_p), ("parents", C.c_void_p),
                    ("k0", C.c_uint32), ("k1", C.c_uint32), ("scheme", C.c_int), ("threshold", C.c_double),
                    ("log_zconst", C.c_double)]

    bufs = dict(x=np.zeros(4 * n), lw=np.zeros(n), w=np.zeros(n), incw=np.zeros(n),
                ctrs=np.zeros(n + 1, np.uint64), counts=np.zeros(n, np.int32), parents=np.zeros(n, np.int32))
    s = Sys(n, *[bufs[k].ctypes.data for k in ("x", "lw", "w", "incw", "ctrs", "counts", "parents")],
            1306, 0, O.SCHEMES[scheme], 0.5, 0.0)
    L.orc_pf_initialize.argtypes = [C.POINTER(Sys), C.c_void_p, C.c_void_p, C.c_int]
    L.orc_pf_step.argtypes = [C.POINTER(Sys), C.c_void_p, C.c_void_p, C.c_int]
    row = np.zeros(5)
    obs = np.ascontiguousarray(obs, np.float64)
    rc = L.orc_pf_initialize(C.byref(s), obs.ctypes.data, row.ctypes.data, threads)
    assert rc == 0
    times = []
    for t in range(1, steps + 1):
        t0 = time.perf_counter()
        rc = L.orc_pf_step(C.byref(s), obs[t % len(obs)].ctypes.data, row.ctypes.data, threads)
        times.append(time.perf_counter() - t0)
        assert rc == 0
    return times


def config1_gpu(P):
    """BASELINE config 1 (the reference's own CPU-runnable case): the paper's PF at N = 10^4,
    100 observations, systematic at ESS < N/2 -- initialize + 99 iterations through the Sampler
    API (CUDA-graph replay on), wall time with a device synchronize on both sides, best of 3
    after one untimed run (which includes the graph capture).  Launch-latency bound."""
    import torch
    obs = bench_obs(100)
    s = P.pf.make_sampler(10000, "systematic", 0.5, seed=1306)
    best = None
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.initialize(obs)
        s.iterate(99)
        s.flush()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if rep:
            best = dt if best is None else min(best, dt)
    return {"workload": "PF config 1: N=10^4, 100 observations, systematic, ESS < N/2 (initialize + 99 "
                        "iterations, CUDA graphs on)", "value": 10000 * 100 / best, "unit": UNIT,
            "us_per_step": best / 100 * 1e6}


def config1_cpu(threads):
    """The C oracle on the same config-1 run: initialize + 99 steps, seconds (wall)."""
    obs = bench_obs(100)
    t0 = time.perf_counter()
    times = cpu_baseline_pf(10000, 99, "systematic", obs, threads)
    return time.perf_counter() - t0, times


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def bench_obs(steps):
    """The synthetic observation track both arms use (T >= 100 rows: the paper's 100-obs shape)."""
    import numpy as np
    return np.cumsum(np.random.default_rng(1306).normal(0, 0.15, (max(100, steps), 2)), 0)


def run_reference(args):
    """--impl reference: the reference algorithm (C oracle port: OpenMP per-particle loops,
    sequential normalization / resampling / copy as SPEC.md:99, :185 pin) on this host's cores,
    on the SAME config as the B200 arm.  Config 2 (N = 2^24) runs at its full N: every timed
    step is one whole PF step of the workload.  Config 4 (2^28 in total) would take ~25 s per
    step on the host, so its steps are bounded samples of 2^24 particles (the rate is per
    particle-step; `sample` says so)."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    n = particles_per_gpu(args, world)
    n_work = n * world
    ns = n_work if n_work <= N_DEFAULT else N_DEFAULT
    # the whole run stays within a few minutes: at ~1.5 s per 2^24 step on 16 host threads, a long
    # --steps (the default 600) takes bounded samples -- the largest power-of-two N whose
    # warmup + steps fit ~150 s (a per-particle-step rate; `same_config` then says false)
    per_ps = 9e-8 * 16 / max(cores, 1)  # host seconds per particle-step (measured: 1.47 s / 2^24 at 16)
    while ns > (1 << 16) and (args.warmup + args.steps) * ns * per_ps > 150.0:
        ns //= 2
    obs = bench_obs(args.steps + args.warmup + 2)
    times = cpu_baseline_pf(ns, args.warmup + args.steps, args.scheme, obs, cores)
    t = sum(times[args.warmup:])
    v = ns * args.steps / t
    scaling, cfg = workload(n, world, args.scheme, is_strong(args, world))
    full = ns == n_work
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup,
            # measured per step at N_s; at the full workload N (config 2) this IS the step time
            "ms_per_step": 1e3 * t / args.steps * (n_work / ns), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg, "same_config": full,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                             "sample": (f"{args.steps} full PF steps of the C oracle at the workload's N={ns} "
                                        if full else
                                        f"{args.steps} full PF steps of the C oracle at N={ns} of the workload's "
                                        f"N={n_work} (rate per particle-step) ") +
                                       f"after {args.warmup} warm-up steps, OpenMP over {cores} threads for the "
                                       "per-particle loops"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU side ---
def run_b200(args):
    import numpy as np
    import torch

    rank, local, world = dist_env()
    # SMC_BENCH_FUNCTIONAL=1: a functional check of the multi-rank path on ONE GPU (every rank on
    # cuda:0, host-staged gloo collectives, so no kernel waits on another rank's kernel).  Its
    # timings are meaningless; the driver's runs use NCCL with one GPU per rank.
    functional = os.environ.get("SMC_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        # NCCL's own INFO log (ranks, rings / NVLS, P2P transport) stays on so the run shows what
        # the communicator set up (stderr; the JSON line stays the last stdout line)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1306_5583_b200 as P

    n = particles_per_gpu(args, world)
    n_total = n * world
    # one GPU: config 2 (N = 2^24); G > 1: config 4 (N = 2^28 in total, 2^28 / G per GPU: strong
    # scaling) unless --particles fixes the per-GPU size (then weak); --config 4 on one GPU: 2^28
    strong = is_strong(args, world)
    T = args.warmup + args.steps + 60  # + the instrumented phase pass
    # synthetic observations of the paper's shape: a smooth track + noise (T x 2)
    obs = bench_obs(T)
    strong_ref = None
    if strong and world > 1 and rank == 0:
        # the same config-4 filter (2^28 particles) on this ONE GPU, timed the same way before the
        # sharded run: the single-GPU point of the strong-scaling curve, inside the same job
        strong_ref = time_single(P, n_total, args, obs)
    if world > 1:
        torch.distributed.barrier()

    shard = None
    if world > 1:  # one rank's slice of a G-GPU filter: global streams, NCCL allgathers + row exchange
        from paper_1306_5583_b200.dist import Shard, TorchComm
        shard = Shard(n, TorchComm())
    s = P.pf.make_sampler(n, args.scheme, 0.5, seed=1306, shard=shard)
    s.initialize(obs)
    s.timing = None
    for _ in range(args.warmup):
        s.iterate(1, check=False)
    s.check()
    torch.cuda.synchronize()
    s.graph = False  # eager launches with PDL (a CUDA-graph replay measured no faster at this N)
    s.timing = None  # no per-phase events inside the timed region (they cost ~25 us per step)
    clk = ClockSampler(local)
    with clk:
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        lc0 = P._abi.launch_count()
        e0.record()
        s.iterate(args.steps, check=False)
        e1.record()
        launches = P._abi.launch_count() - lc0  # the library's own kernels in the timed region
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    s.check()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    h = s.history()
    resampled = h["resampled"][-args.steps:]
    prev_rs = h["resampled"][-args.steps - 1:-1]
    # phase breakdown from a separate, instrumented pass (per-phase CUDA events), outside the timed region
    s.timing = {}
    s.iterate(min(args.steps, 50), check=False)
    torch.cuda.synchronize()
    # per-phase medians over the instrumented steps (robust to a stray slow step, e.g. a clock
    # ramp right after the timed region); the full lists go to stderr for inspection
    phase_lists = {k: sorted(a.elapsed_time(b) for a, b in v) for k, v in s.timing.items()}
    phase = {k: v[len(v) // 2] for k, v in phase_lists.items()}
    print(json.dumps({"phase_ms_sorted": phase_lists}), file=sys.stderr)
    s.timing = None

    # ---- roofline of the dominant kernel (the fused move) and of resample+copy ----
    peak, peak_src = measured_peaks()
    # X 32 R + 32 W, lw 8 W; + the parent index (4 R) after a resample, else lw 8 R; the
    # counters (8 R + 8 W) only when the streams are not at one uniform count (smc_pf_move_uniform)
    uni = s.system.rng_set.uniform_count(s.system.size, 16) is not None
    move_bytes = n * (32 + 32 + 8 + (0 if uni else 16)) + n * (4 * float(np.mean(prev_rs)) + 8 * float(np.mean(1 - prev_rs)))
    move_gbs = move_bytes / (phase["move"] * 1e-3) / 1e9
    # resample+copy (the metric's second half, SURVEY §8d config 5 at this N): smc_resample with the
    # parent map AND the explicit in-place row copy, timed alone with CUDA events (inside the PF step
    # the copy is folded into the next move's gather instead).  Algorithmic bytes: W 8 R + counts 4 W
    # + parents 4 W per particle + 64 B per moved 32-byte row.  The weights are the same whatever
    # --steps is: a fresh filter (same seed and track) run for the paper's 100 observations, the last
    # move taken without its resample -- the PF's real pre-resample weight distribution at t = 100.
    s_rc = P.pf.make_sampler(n, args.scheme, 0.5, seed=1306, shard=shard)
    s_rc.initialize(obs)
    s_rc.iterate(98, check=False)
    s_rc.move_queue[0](s_rc.iteration + 1, s_rc.system)
    rc = resample_copy_bench(P, s_rc.system, args.scheme)
    del s_rc
    torch.cuda.empty_cache()
    frac_moved = rc["moved_frac"]
    dominant = max(("move", "resample", "monitor"), key=lambda k: phase.get(k, 0))

    value = n_total * args.steps / (ms * 1e-3)
    scaling, cfg = workload(n, world, args.scheme, strong)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "l2": f"inputs larger than L2 (state {32 * n >> 20} MiB per GPU), no flush",
            "parallelism": f"particles sharded over {world} GPU(s)",
            "phase_ms": phase, "resampled_frac": float(np.mean(resampled)), "moved_row_frac": frac_moved,
            # counted by the library (smc_launch_count) around the timed iterate(): per step the move,
            # the lse combine, the ESS rule, the device-gated resample passes and set_equal_weight
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": "k_pf_move (fused move + add_log_weight + lse/ESS partials)",
                         "achieved": move_gbs, "peak": peak, "unit": "GB/s", "frac": move_gbs / peak,
                         "traffic": move_traffic(n), "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": move_bytes,
                         # the kernel is compute-bound by the reference's RNG contract:
                         # its issue floor from the ncu instruction count, against the measured time
                         "compute": compute_floor(n, phase["move"])},
            "resample_copy": {"achieved": rc["gbs"], "peak": peak, "unit": "GB/s", "frac": rc["gbs"] / peak,
                              "ms": rc["ms"], "algorithmic_bytes": rc["bytes"], "scheme": args.scheme,
                              "weights": "the PF's pre-resample weights at t = 100 (fresh filter, same seed)",
                              "reps": rc["reps"],
                              "kernels": "k_rs_tiles, k_rs_scan, k_rs_counts, k_rs_zsp_scan, k_rs_ranks, "
                                         "k_rs_assign<copy fused>"},
            "dominant_phase": dominant, "clocks": clk.summary()}

    # ---- e2e: the public API with host buffers: per step H2D the observation pair from pinned
    # memory and D2H the step's history row (ess/N, resampled, pos.0, pos.1) ----
    if not args.no_e2e:
        e = run_e2e(P, s, obs, args.steps)
        line["e2e"] = {"value": n_total * args.steps / e["seconds"], "unit": UNIT,
                       "h2d_bytes_per_step": e["h2d"], "d2h_bytes_per_step": e["d2h"]}
    if rank == 0 and world == 1 and not args.no_gmm:
        line["gmm"] = gmm_bench(P)
    if strong_ref is not None:
        line["strong_baseline"] = dict(strong_ref, note="the same config-4 filter on ONE GPU of this job "
                                       "(rank 0, before the sharded run): strong-scaling efficiency at "
                                       f"{world} GPUs = value / (strong_baseline.value * {world})")
    if rank == 0 and world == 1 and not args.no_schemes and args.n is None and config_of(args, world) == 2:
        line["schemes"] = schemes_bench(P, n, args, obs)
    if rank == 0 and world == 1 and not args.no_config1:
        line["config1"] = config1_gpu(P)
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_line(n, args.scheme, obs)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def time_single(P, n, args, obs):
    """One unsharded filter of n particles on this GPU: ms per step over args.steps (CUDA events)."""
    import torch
    s = P.pf.make_sampler(n, args.scheme, 0.5, seed=1306)
    s.initialize(obs)
    for _ in range(args.warmup):
        s.iterate(1, check=False)
    s.check()
    s.graph = False
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.iterate(args.steps, check=False)
    e1.record()
    torch.cuda.synchronize()
    s.check()
    ms = e0.elapsed_time(e1)
    del s
    torch.cuda.empty_cache()
    return {"value": n * args.steps / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms / args.steps, "n_particles": n,
            "n_gpus": 1}


def schemes_bench(P, n, args, obs, steps=30, warmup=3):
    """Config 2's sweep: the 2^24 PF step (move + ESS + resample + parent map + fused copy) for
    every resampling scheme, eager launches timed with CUDA events over `steps` steps."""
    import numpy as np
    import torch
    out = {}
    for scheme in ("multinomial", "residual", "stratified", "systematic", "residual_stratified",
                   "residual_systematic"):
        s = P.pf.make_sampler(n, scheme, 0.5, seed=1306)
        s.initialize(obs)
        for _ in range(warmup):
            s.iterate(1, check=False)
        s.graph = False
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.iterate(steps, check=False)
        e1.record()
        torch.cuda.synchronize()
        s.check()
        ms = e0.elapsed_time(e1) / steps
        h = s.history()
        out[scheme] = {"ms_per_step": ms, "value": n / (ms * 1e-3), "unit": UNIT,
                       "resampled_frac": float(np.mean(h["resampled"][-steps:]))}
        del s
        torch.cuda.empty_cache()
    return out


def cpu_baseline_line(n, scheme, obs):
    """The oracle on this box's host cores at the workload's own N: 3 timed steps with all cores
    (OpenMP per-particle loops) and 1 timed step on one thread (the sequential figure)."""
    cores = len(os.sched_getaffinity(0))
    tm = cpu_baseline_pf(n, 4, scheme, obs, cores)[1:]  # first step untimed (page faults)
    t1 = cpu_baseline_pf(n, 1, scheme, obs, 1)
    v = n * len(tm) / sum(tm)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"{len(tm)} full PF steps of the C oracle at the workload's N={n} (after 1 untimed step), "
                      f"OpenMP over {cores} threads for the per-particle loops",
            "sequential": {"value": n / t1[0], "unit": UNIT, "cores": 1,
                           "sample": f"1 full PF step of the C oracle at N={n} on one thread"},
            "config1": {f"cores_{c}": {"value": 10000 * 100 / config1_cpu(c)[0], "unit": UNIT, "cores": c}
                        for c in sorted({1, cores})} | {
                "sample": "config 1 in full: the C oracle's initialize + 99 PF steps at N=10^4 (wall)"}}


def gmm_bench(P, n=1 << 20, T=100):
    """BASELINE config 3 alongside the PF line: the GMM SMC sampler (4 components, 1000 synthetic
    points, prior annealing p = 2, T = 100, N = 2^20), initialize + iterate timed with CUDA events.
    FP64-issue bound (3 MH blocks x 1000 points x 4 components per particle-iteration)."""
    import torch
    from paper_1306_5583_b200 import gmm
    y = gmm.generate_data(1000, 1306)
    w = gmm.make_sampler(4096, data=y, T=5, seed=1)  # warm-up (module load, first launches)
    w.initialize()
    w.iterate(5)
    s = gmm.make_sampler(n, data=y, T=T, seed=1307)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.initialize()
    s.iterate(T)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    evals = n * 3 * T * 1000 * 4  # (particle, point, component) likelihood terms in the 3T MH blocks
    out = {"workload": "GMM config 3: N=2^20, 4 components, 1000 points, T=100, prior annealing p=2",
           "value": n * T / (ms * 1e-3), "unit": "particle-iterations/s", "ms_per_run": ms,
           "log_zconst_ds": s.log_zconst, "log_zconst_ps": s.path_log_zconst(),
           "component_evals_per_s": n * (1 + 3 * T) * 1000 * 4 / (ms * 1e-3)}
    # FP64 roofline: fp64 thread-instructions per likelihood term from the committed ncu capture of
    # one k_gmm_mh launch (stamped with the kernel sources), times the terms of the whole run, over
    # the run's time, against the fp64 pipe's issue rate (64 lanes / SM / clk x 148 SMs x max clock)
    d, src = profile_for("gmm_mh_ncu", n)
    if d is not None:
        per = d["fp64_thread_inst"] / (d["n"] * d["nd"] * d["r"])
        ach = per * evals / (ms * 1e-3)
        peak = 64 * 148 * 1.965e9
        out["fp64"] = {"bound": "fp64 pipe", "fp64_inst_per_term": per, "achieved_inst_per_s": ach,
                       "peak_inst_per_s": peak, "frac": ach / peak,
                       "ncu_fp64_pipe_pct_one_launch": d.get("fp64_pipe_pct"), "source": src}
    else:
        out["fp64"] = {"frac": None, "source": src}
    return out


def source_hash():
    """The library's source stamp (every csrc/ file + the ABI header + the nvcc flags)."""
    from paper_1306_5583_b200 import _build
    return _build.source_hash()


def profile_for(name, n):
    """A committed ncu capture (profiles/<name>.json) -- used only when it was taken at this N AND
    from the current kernel sources (its `source_hash`): a kernel change never reuses a stale
    capture silently; the field reads null with the reason instead."""
    try:
        with open(os.path.join(ROOT, "profiles", name + ".json")) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None, f"profiles/{name}.json missing"
    if d.get("n") != n:
        return None, f"profiles/{name}.json taken at N={d.get('n')}"
    if d.get("source_hash") != source_hash():
        return None, f"profiles/{name}.json is from other kernel sources (commit {d.get('commit')}): re-capture"
    return d, f"profiles/{name}.json (ncu --set full, commit {d.get('commit')}, same source hash)"


def move_traffic(n):
    """DRAM bytes (read + write) per k_pf_move launch from the committed ncu capture, or None."""
    d, _ = profile_for("move_ncu", n)
    return None if d is None else d["dram_bytes_read"] + d["dram_bytes_write"]


def compute_floor(n, move_ms):
    """Issue floor of k_pf_move: instructions per particle (ncu) over 148 SMs x 4 schedulers x 32
    lanes at the max SM clock -- the compute roofline the move is held to."""
    d, src = profile_for("move_ncu", n)
    if d is None:
        return {"frac": None, "source": src}
    ipp = d["warp_inst_per_particle"] * 32.0 if "warp_inst_per_particle" in d else d["inst_per_particle"]
    floor_ms = n * ipp / (148 * 128 * 1.965e9) * 1e3
    return {"bound": "issue (IMAD.WIDE Philox on the FMA pipe + fp64 Box-Muller)", "instr_per_particle": ipp,
            "issue_floor_ms": floor_ms, "achieved_ms": move_ms, "frac": floor_ms / move_ms, "source": src}


def resample_copy_bench(P, system, scheme, reps=10):
    """smc_resample (counts + parents + in-place 32-byte row copy) on the system's current
    normalized weights and a scratch copy of its state; mean ms over `reps` calls."""
    import ctypes

    import torch
    from paper_1306_5583_b200 import _abi
    n = system.size
    w = system.weight_set.read_weight()
    if system.shard is not None:  # a shard's weights sum to its share of the global mass
        w = w / w.sum()
    w = w.contiguous()
    x = system.value.data.clone()
    counts = torch.empty(n, dtype=torch.int32, device="cuda")
    parents = torch.empty(n, dtype=torch.int32, device="cuda")
    status = torch.zeros(3, dtype=torch.int32, device="cuda")  # smc_status
    ws = torch.empty(_abi.lib().smc_resample_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    rng = P.RngStreamSet(n + 1, 1306)
    from paper_1306_5583_b200.resample import _scheme
    sid = int(_scheme(scheme))

    def call():
        _abi.call("smc_resample", sid, _abi.ptr(w), None, None, n, n, rng.seed, n, rng.counter_ptr(n), None, 0,
                  _abi.ptr(counts), _abi.ptr(parents), ctypes.c_void_p(x.data_ptr()), 32, None, _abi.ptr(status),
                  _abi.ptr(ws), ws.numel(), _abi.stream())
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    if int(status[0].item()) != 0:
        raise RuntimeError(f"resample+copy bench: device status {int(status[0].item())}")
    ms = e0.elapsed_time(e1) / reps
    moved = int((parents != torch.arange(n, device="cuda", dtype=torch.int32)).sum().item())
    byts = n * (8 + 4 + 4) + 64 * moved
    del x, ws
    return {"ms": ms, "bytes": byts, "gbs": byts / (ms * 1e-3) / 1e9, "moved_frac": moved / n, "reps": reps}


def run_e2e(P, s, obs, steps):
    """Same steps through Sampler with host-resident inputs/outputs, copies inside the timed region."""
    import numpy as np
    import torch

    value = s.system.value
    dev_obs = value.obs
    host_obs = torch.from_numpy(np.ascontiguousarray(obs)).pin_memory()
    ncols = len(s._cols)
    host_rows = torch.empty((steps + 1, ncols), dtype=torch.float64).pin_memory()
    # re-initialize so iteration indices line up with the host observation buffer
    s.initialize(obs)
    torch.cuda.synchronize()
    hist = s._hist
    stream = torch.cuda.current_stream()
    # the copies run on their own stream, ordered against the steps by events: step t's
    # observation is uploaded while step t-1 computes, and record t-1 is read back while step
    # t+1 computes -- the per-step transfers stay inside the timed region, off the step chain
    copy = torch.cuda.Stream()
    done = [None] * (steps + 1)
    h2d = [None] * (steps + 1)
    t0 = time.perf_counter()
    t1 = s.iteration + 1
    with torch.cuda.stream(copy):
        dev_obs[t1].copy_(host_obs[t1], non_blocking=True)  # H2D: step 1's observation (16 B)
        h2d[0] = torch.cuda.Event()
        h2d[0].record(copy)
    for k in range(steps):
        t = s.iteration + 1
        stream.wait_event(h2d[k])
        s.iterate(1, check=False)
        stepped = torch.cuda.Event()
        stepped.record(stream)
        with torch.cuda.stream(copy):
            if k + 1 < steps:  # H2D: the next step's observation (16 B), while this step computes
                dev_obs[t + 1].copy_(host_obs[t + 1], non_blocking=True)
                h2d[k + 1] = torch.cuda.Event()
                h2d[k + 1].record(copy)
            # D2H: the newest COMPLETE history record.  The "pos" monitor of step t is
            # reduced by step t+1's move (fused), so each step reads record t-1; the
            # last record is flushed and read after the loop, inside the timed region.
            copy.wait_event(stepped)
            host_rows[k].copy_(s._hist[t - 1], non_blocking=True)
            done[k] = torch.cuda.Event()
            done[k].record(copy)
        if k:  # streaming consumer: step k-1's record is in host memory before step k+1 is issued
            done[k - 1].synchronize()
    host_rows[steps].copy_(s.history_row(s.iteration), non_blocking=True)
    stream.synchronize()
    copy.synchronize()
    sec = time.perf_counter() - t0
    del hist
    s.check()
    return {"seconds": sec, "h2d": 16, "d2h": 8 * ncols}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
