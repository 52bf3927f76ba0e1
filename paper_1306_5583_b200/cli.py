"""Command-line entry point (mirror of smckit's cli module).

    python -m paper_1306_5583_b200 pf  --data pf.data|simulate --particles 1000 --seed 7 --out pf.est
    python -m paper_1306_5583_b200 gmm --components 4 --particles 8192 --iters 100 --anneal prior:2 \
        --seed 7 --data simulate --out gmm.est
    python -m paper_1306_5583_b200 bench --min-log2 3 --max-log2 17 --out bench.tsv
    python -m paper_1306_5583_b200 generate pf|gmm --seed 1306 --out pf.data

Every output file starts with comment lines holding the fully resolved config
(RunConfig); re-running with those values reproduces the file
byte for byte (the whole path is deterministic, GPU included).
TSVs use tabs and 17 significant digits.  Exit codes: 0 success,
1 usage, 2 runtime failure.  The backend is the CUDA grid
(``--backend cuda``); the reference's seq / pool:k backends do not exist here.
"""

from __future__ import annotations

import argparse
import sys
import time

import numpy as np

__all__ = ["main", "load_gmm_data", "write_gmm_data"]

SCHEMES = {"multinomial": "Multinomial", "residual": "Residual", "stratified": "Stratified",
           "systematic": "Systematic", "residual_stratified": "ResidualStratified",
           "residual_systematic": "ResidualSystematic"}


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage problems exit 1, not argparse's 2
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(1)


def load_gmm_data(path):
    """One float per line; '#' comments and blank lines skipped;
    a malformed line raises ValueError naming its line number."""
    vals = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            parts = s.split()
            if len(parts) != 1:
                raise ValueError(f"{path}:{ln}: expected 1 value, got {len(parts)}")
            try:
                vals.append(float(parts[0]))
            except ValueError as e:
                raise ValueError(f"{path}:{ln}: {e}") from None
    return np.asarray(vals, dtype=np.float64)


def write_gmm_data(path, y):
    with open(path, "w") as f:
        for v in y:
            f.write(f"{v:.17g}\n")


def _scheme(name):
    from .resample import ResampleScheme
    key = name.lower().replace("-", "_")
    if key not in SCHEMES:
        raise UsageError(f"unknown scheme {name!r} (one of {', '.join(SCHEMES)})")
    return getattr(ResampleScheme, SCHEMES[key])


def _anneal(spec):
    """'linear' or 'prior:p' -> power (1 = linear)."""
    if spec == "linear":
        return 1.0
    if spec.startswith("prior"):
        p = spec.split(":", 1)[1] if ":" in spec else "2"
        try:
            p = float(p)
        except ValueError:
            raise UsageError(f"bad --anneal {spec!r}") from None
        if not p > 1:
            raise UsageError("prior annealing needs p > 1 (SPEC.md:578)")
        return p
    raise UsageError(f"bad --anneal {spec!r} (linear | prior:p)")


def _backend(b):
    if b != "cuda":
        raise UsageError(f"backend {b!r} unavailable: the CUDA grid replaces seq / pool:k (exec, SPEC.md:388-391)")


def _header(cmd, cfg):
    lines = [f"smc_b200 {cmd}"]
    lines += [f"{k}={cfg[k]}" for k in sorted(cfg)]
    return lines


def _write(path, text):
    if path == "-":
        sys.stdout.write(text)
    else:
        with open(path, "w") as f:
            f.write(text)


# --------------------------------------------------------------------------- pf
def cmd_pf(a):
    from . import pf
    _backend(a.backend)
    scheme = _scheme(a.scheme)
    if a.particles < 1:
        raise UsageError("--particles must be >= 1")
    if a.data == "simulate":
        obs, _ = pf.generate_observations(a.n_data, a.data_seed)
    else:
        obs = pf.load_observations(a.data)
    cfg = {"particles": a.particles, "seed": a.seed, "scheme": a.scheme, "threshold": repr(a.threshold),
           "data": a.data, "backend": a.backend}
    if a.data == "simulate":
        cfg.update({"n_data": a.n_data, "data_seed": a.data_seed})
    s = pf.make_sampler(a.particles, scheme, a.threshold, a.seed)
    s.initialize(obs)
    s.iterate(obs.shape[0] - 1)
    text = s.write_tsv(_NullIO(), header_comments=_header("pf", cfg))
    _write(a.out, text)
    print(f"log_zconst\t{s.log_zconst:.17g}")
    return 0


# -------------------------------------------------------------------------- gmm
def cmd_gmm(a):
    from . import gmm
    _backend(a.backend)
    scheme = _scheme(a.scheme)
    power = _anneal(a.anneal)
    if a.particles < 1 or a.iters < 1:
        raise UsageError("--particles and --iters must be >= 1")
    if not 1 <= a.components <= gmm.MAX_R:
        raise UsageError(f"--components must be in [1, {gmm.MAX_R}]")
    y = gmm.generate_data(a.n_data, a.data_seed) if a.data == "simulate" else load_gmm_data(a.data)
    if y.size == 0:
        raise ValueError(f"{a.data}: no observations")
    hyper = gmm.default_hyper(y, a.lambda_known)
    if a.hyper:
        try:
            vals = [float(v) for v in a.hyper.split(",")]
        except ValueError:
            raise UsageError(f"bad --hyper {a.hyper!r}") from None
        if len(vals) != 5:
            raise UsageError("--hyper takes xi,kappa,nu,chi,rho")
        hyper = vals + [a.lambda_known]
    cfg = {"components": a.components, "particles": a.particles, "iters": a.iters, "anneal": a.anneal,
           "seed": a.seed, "scheme": a.scheme, "threshold": repr(a.threshold), "data": a.data,
           "hyper": ",".join(repr(float(v)) for v in hyper[:5]), "lambda_known": repr(a.lambda_known),
           "backend": a.backend}
    if a.data == "simulate":
        cfg.update({"n_data": a.n_data, "data_seed": a.data_seed})
    s = gmm.make_sampler(a.particles, data=y, T=a.iters, power=power, scheme=scheme, threshold=a.threshold,
                         seed=a.seed, hyper=hyper, components=a.components)
    s.initialize()
    s.iterate(a.iters)
    ds, ps = s.log_zconst, s.path_log_zconst()
    text = s.write_tsv(_NullIO(), header_comments=_header("gmm", cfg) + [f"ds_log_zconst={ds!r}",
                                                                          f"ps_log_zconst={ps!r}"])
    _write(a.out, text)
    print(f"ds_log_zconst\t{ds:.17g}")
    print(f"ps_log_zconst\t{ps:.17g}")
    return 0


# ------------------------------------------------------------------------ bench
def cmd_bench(a):
    """the GMM sampler over N = 2^min .. 2^max, wall-clock seconds of
    initialize + iterate (data loading excluded), median of --reps repetitions.  One
    backend exists (the CUDA grid), so the speedup column is relative to the first N's
    per-particle cost: particle-iterations/s at N over that at 2^min."""
    import torch
    from . import gmm, pf
    _backend(a.backend)
    if a.min_log2 < 0 or a.max_log2 < a.min_log2 or a.max_log2 > 30:
        raise UsageError("need 0 <= --min-log2 <= --max-log2 <= 30")
    if a.model == "gmm":
        y = gmm.generate_data(a.n_data, a.data_seed)
    else:
        obs, _ = pf.generate_observations(pf.DATA_NUM, a.data_seed)
    cfg = {"model": a.model, "iters": a.iters, "reps": a.reps, "seed": a.seed, "min_log2": a.min_log2,
           "max_log2": a.max_log2, "backend": a.backend, "n_data": a.n_data, "data_seed": a.data_seed}
    rows, base = [], None
    for lg in range(a.min_log2, a.max_log2 + 1):
        n = 1 << lg
        times = []
        for rep in range(a.reps + 1):  # rep 0: warm-up (module load, allocation)
            if a.model == "gmm":
                s = gmm.make_sampler(n, data=y, T=a.iters, seed=a.seed + rep)
                steps = a.iters
            else:
                s = pf.make_sampler(n, seed=a.seed + rep)
                steps = min(a.iters, obs.shape[0] - 1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if a.model == "gmm":
                s.initialize()
            else:
                s.initialize(obs)
            s.iterate(steps)
            s.flush()
            torch.cuda.synchronize()
            if rep:
                times.append(time.perf_counter() - t0)
        med = float(np.median(times))
        rate = n * steps / med
        base = base or rate
        rows.append((n, med, rate, rate / base))
        print(f"N=2^{lg}\t{med:.6f} s\t{rate:.4g} particle-iterations/s", file=sys.stderr)
    lines = [f"# {c}" for c in _header("bench", cfg)]
    lines.append("\t".join(["particles", "cuda_seconds", "particle_iterations_per_s", "speedup_vs_min_n"]))
    for n, med, rate, sp in rows:
        lines.append(f"{n}\t{med:.17g}\t{rate:.17g}\t{sp:.17g}")
    _write(a.out, "\n".join(lines) + "\n")
    return 0


# --------------------------------------------------------------------- generate
def cmd_generate(a):
    if a.model == "pf":
        from . import pf
        obs, truth = pf.generate_observations(a.n or pf.DATA_NUM, a.seed)
        pf.write_observations(a.out, obs, truth)  # + .truth sibling
    else:
        from . import gmm
        write_gmm_data(a.out, gmm.generate_data(a.n or 100, a.seed))
    return 0


class _NullIO:
    def write(self, _):
        pass


def build_parser():
    p = _Parser(prog="python -m paper_1306_5583_b200", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    def common(q, particles, out):
        q.add_argument("--particles", type=int, default=particles)
        q.add_argument("--seed", type=int, default=0)
        q.add_argument("--backend", default="cuda")
        q.add_argument("--threshold", type=float, default=0.5)
        q.add_argument("--data", default="simulate", help="file path or 'simulate'")
        q.add_argument("--data-seed", type=int, default=1306)
        q.add_argument("--out", default=out)

    q = sub.add_parser("pf", help="particle filter (SPEC.md:510)")
    common(q, 1000, "pf.est")
    q.add_argument("--scheme", default="systematic")
    q.add_argument("--n-data", type=int, default=100)
    q.set_defaults(fn=cmd_pf)

    q = sub.add_parser("gmm", help="GMM SMC sampler (SPEC.md:601)")
    common(q, 8192, "gmm.est")
    q.add_argument("--components", type=int, default=4)
    q.add_argument("--iters", type=int, default=100)
    q.add_argument("--anneal", default="prior:2")
    q.add_argument("--scheme", default="stratified")
    q.add_argument("--n-data", type=int, default=100)
    q.add_argument("--hyper", default=None, help="xi,kappa,nu,chi,rho (default: SPEC.md:592)")
    q.add_argument("--lambda-known", type=float, default=0.0)
    q.set_defaults(fn=cmd_gmm)

    q = sub.add_parser("bench", help="timings over N (SPEC.md:634-638)")
    q.add_argument("--model", choices=["gmm", "pf"], default="gmm")
    q.add_argument("--min-log2", type=int, default=3)
    q.add_argument("--max-log2", type=int, default=17)
    q.add_argument("--iters", type=int, default=100)
    q.add_argument("--reps", type=int, default=5)
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--backend", default="cuda")
    q.add_argument("--n-data", type=int, default=100)
    q.add_argument("--data-seed", type=int, default=1306)
    q.add_argument("--out", default="bench.tsv")
    q.set_defaults(fn=cmd_bench)

    q = sub.add_parser("generate", help="write synthetic data (SPEC.md:641-647)")
    q.add_argument("model", choices=["pf", "gmm"])
    q.add_argument("--seed", type=int, default=1306)
    q.add_argument("--n", type=int, default=0)
    q.add_argument("--out", required=True)
    q.set_defaults(fn=cmd_generate)
    return p


def main(argv=None):
    p = build_parser()
    a = p.parse_args(argv)
    try:
        return a.fn(a)
    except UsageError as e:
        p.print_usage(sys.stderr)
        sys.stderr.write(f"error: {e}\n")
        return 1
    except (OSError, ValueError, RuntimeError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
