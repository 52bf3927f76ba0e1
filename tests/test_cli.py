"""CLI: usage errors, data files, provenance and determinism."""

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_1306_5583_b200", *args], capture_output=True, text=True,
                          cwd=cwd or ROOT, timeout=600)


def test_unknown_flag_is_usage_error():
    r = _run("pf", "--no-such-flag")
    assert r.returncode == 1 and "usage" in r.stderr.lower()


def test_unknown_subcommand():
    assert _run("nope").returncode == 1


def test_backend_and_anneal_validation():
    from paper_1306_5583_b200 import cli
    with pytest.raises(cli.UsageError):
        cli._backend("pool:4")
    assert cli._anneal("linear") == 1.0 and cli._anneal("prior:3") == 3.0 and cli._anneal("prior") == 2.0
    with pytest.raises(cli.UsageError):
        cli._anneal("prior:0.5")
    with pytest.raises(cli.UsageError):
        cli._scheme("bogus")
    assert cli._scheme("residual-systematic").name == "ResidualSystematic"


def test_gmm_data_roundtrip_and_errors(tmp_path):
    from paper_1306_5583_b200 import cli
    y = np.array([0.1, -2.5, 1e-300, 3.141592653589793, 7.0])
    p = tmp_path / "g.data"
    cli.write_gmm_data(p, y)
    assert np.array_equal(cli.load_gmm_data(p), y)  # full precision
    bad = tmp_path / "bad.data"
    bad.write_text("1.0\n2.0 3.0\n")
    with pytest.raises(ValueError, match=":2:"):
        cli.load_gmm_data(bad)  # error names the line
    bad.write_text("1.0\nx\n")
    with pytest.raises(ValueError, match=":2:"):
        cli.load_gmm_data(bad)


def test_pf_data_errors(tmp_path):
    from paper_1306_5583_b200 import pf
    bad = tmp_path / "pf.data"
    bad.write_text("1 2\n3\n")
    with pytest.raises(ValueError, match=":2:"):
        pf.load_observations(bad)


def test_missing_data_file_exit_2(tmp_path):
    r = _run("gmm", "--data", str(tmp_path / "missing.data"), "--out", str(tmp_path / "o.est"))
    assert r.returncode in (1, 2) and "error" in r.stderr


@pytest.mark.gpu
def test_pf_cli_deterministic(tmp_path):
    a, b = tmp_path / "a.est", tmp_path / "b.est"
    for out in (a, b):
        r = _run("pf", "--particles", "1000", "--seed", "7", "--out", str(out))
        assert r.returncode == 0, r.stderr
    assert a.read_bytes() == b.read_bytes()
    text = a.read_text().splitlines()
    assert text[0] == "# smc_b200 pf" and any(l == "# seed=7" for l in text)
    hdr = [l for l in text if not l.startswith("#")][0].split("\t")
    assert hdr[:3] == ["iter", "ess_over_n", "resampled"] and hdr[-2:] == ["pos.0", "pos.1"]
    assert len([l for l in text if not l.startswith("#")]) == 101


@pytest.mark.gpu
def test_gmm_cli_and_generate(tmp_path):
    d = tmp_path / "g.data"
    assert _run("generate", "gmm", "--seed", "5", "--n", "80", "--out", str(d)).returncode == 0
    out = tmp_path / "gmm.est"
    r = _run("gmm", "--components", "2", "--particles", "2048", "--iters", "20", "--anneal", "linear",
             "--seed", "3", "--data", str(d), "--out", str(out))
    assert r.returncode == 0, r.stderr
    vals = dict(l.split("\t") for l in r.stdout.strip().splitlines())
    assert set(vals) == {"ds_log_zconst", "ps_log_zconst"}
    ds, ps = float(vals["ds_log_zconst"]), float(vals["ps_log_zconst"])
    assert np.isfinite(ds) and np.isfinite(ps)
    text = out.read_text()
    assert f"# ds_log_zconst={ds!r}" in text and "# components=2" in text
    cols = [l for l in text.splitlines() if not l.startswith("#")][0].split("\t")
    assert cols == ["iter", "ess_over_n", "resampled", "accept.0", "accept.1", "accept.2", "accept.3", "path.grid",
                    "path.integrand"]  # accept.0: the move queue; 1-3: mu, lambda, weight blocks
    r2 = _run("gmm", "--components", "2", "--particles", "2048", "--iters", "20", "--anneal", "linear",
              "--seed", "3", "--data", str(d), "--out", str(tmp_path / "again.est"))
    assert (tmp_path / "again.est").read_bytes() == out.read_bytes()


@pytest.mark.gpu
def test_bench_cli(tmp_path):
    out = tmp_path / "bench.tsv"
    r = _run("bench", "--min-log2", "3", "--max-log2", "5", "--iters", "5", "--reps", "2", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rows = [l for l in out.read_text().splitlines() if not l.startswith("#")]
    assert rows[0].split("\t")[0] == "particles" and [int(l.split("\t")[0]) for l in rows[1:]] == [8, 16, 32]
