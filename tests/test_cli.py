"""csrc_bench CLI (paper_1003_0952_b200/csrc/cli.cpp), the counterpart of the
reference's bench tool (tools/bench_main.cpp): run / verify / info with the
same flags, messages and report fields (BenchReport, bench.hpp:24-55).
CPU tests cover argument handling and Matrix Market ingestion errors (raised
before any device call); GPU tests the subcommands end to end."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import Ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1003_0952_b200", "csrc_bench")
FIELDS = ["matrix", "n", "nnz_stored", "nnz_full", "nnz_per_row", "ws_kb", "format", "strategy", "accum", "p",
          "reps", "runs", "median_total_seconds", "mflops_effective", "mflops_true", "speedup_vs_seq_csrc",
          "init_max", "compute_max", "accumulate_max", "n_colors"]


def cli(*args, timeout=300):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout)


def test_cli_built():
    assert os.access(CLI, os.X_OK), "csrc_bench missing: make -C paper_1003_0952_b200/csrc"


def test_usage_errors():
    r = cli()
    assert r.returncode == 2 and "a subcommand is required" in r.stderr
    r = cli("info")
    assert r.returncode == 2 and r.stderr.strip() == "error: one of --matrix or --gen is required"
    r = cli("run", "--gen", "band:n=5", "--strategy", "bogus")
    assert r.returncode == 2 and "--strategy" in r.stderr
    r = cli("run", "--gen", "band:n=5", "--reps", "0")
    assert r.returncode == 2 and "--reps" in r.stderr
    r = cli("info", "--gen", "band:n=5", "--matrix", "x.mtx")
    assert r.returncode == 2 and "exclude" in r.stderr
    r = cli("info", "--matrix", "/nonexistent/a.mtx")
    assert r.returncode == 1 and r.stderr.strip() == "error: cannot open '/nonexistent/a.mtx'"


@pytest.mark.parametrize("text,msg", [
    ("", "matrix market: empty stream"),
    ("%%MatrixMarket matrix array real general\n2 2\n", "matrix market, line 1: only coordinate format is supported"),
    ("%%MatrixMarket matrix coordinate complex general\n", "matrix market, line 1: unsupported field 'complex'"),
    ("%%MatrixMarket matrix coordinate real hermitian\n", "matrix market, line 1: unsupported symmetry 'hermitian'"),
    ("%%MatrixMarket matrix coordinate real general\n% c\n2 x 1\n", "matrix market, line 3: malformed size line '2 x 1'"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "matrix market, line 3: expected 2 entries, got 1"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
     "matrix market, line 3: index (3, 1) outside declared bounds"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "matrix market, line 3: missing value in '1 1'"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n1 1 2.0\n",
     "matrix market, line 3: skew-symmetric file stores a diagonal entry"),
])
def test_matrix_market_errors(tmp_path, text, msg):
    """matrix_market.hpp:15-85 wording, line numbers counted the same way."""
    p = tmp_path / "m.mtx"
    p.write_text(text)
    r = cli("info", "--matrix", str(p))
    assert r.returncode == 1 and r.stderr.strip() == "error: " + msg


def write_mtx(path, n, rows, cols, vals, sym="general"):
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate real {sym}\n% test\n{n} {n} {len(rows)}\n")
        for r, c, v in zip(rows, cols, vals):
            f.write(f"{r + 1} {c + 1} {v!r}\n")


@pytest.mark.gpu
@pytest.mark.parametrize("gen", ["band:n=300,h=3", "band:n=200,h=5,valsym=1", "random_sym:n=400,density=0.03,seed=5",
                                 "dense:n=40", "random_sym:n=2500,density=0.004,seed=2"])
def test_verify_passes(gen):
    r = cli("verify", "--gen", gen, "--threads", "1,2,4")
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "VERIFY PASS"
    assert any(l.startswith("pass  seq csrc p=1") for l in lines)
    assert sum(l.startswith("pass  buffers/") for l in lines) == 12
    assert sum(l.startswith("pass  colorful p=") for l in lines) == 3


@pytest.mark.gpu
def test_verify_detects_corrupted_coloring():
    r = cli("verify", "--gen", "band:n=50,h=2", "--strategy", "colorful", "--threads", "2", "--corrupt-coloring")
    assert r.returncode == 1
    assert "FAIL  colorful p=2" in r.stdout and "coloring violation: rows" in r.stdout
    assert r.stdout.strip().endswith("VERIFY FAIL")


@pytest.mark.gpu
def test_info_matches_reference_matrix_info(tmp_path):
    """info prints matrix_info (bench.hpp:113-122): name, value symmetric,
    n, nnz (stored convention), nnz/n, ws_kb (floored working_set_kb)."""
    R = Ref()
    for gen, (n, dens, seed, vs) in {"random_sym": (300, 0.05, 9, 0)}.items():
        r, c, v = R.gen_random_sym(n, dens, seed, bool(vs))
        ref = R.build_csrc(n, r, c, v)
        k = ref["ja"].size
        nnz = n + 2 * k  # not value symmetric: full count
        ws = int(R.lib.ref_working_set_kb(n, nnz, 0))
        out = cli("info", "--gen", f"random_sym:n={n},density={dens},seed={seed}")
        assert out.returncode == 0, out.stderr
        assert out.stdout.split() == ["random_sym", "no", str(n), str(nnz), str(nnz // n), str(ws)]
    out = cli("info", "--gen", "band:n=100,h=2,valsym=1")
    n, k = 100, 2 * 100 - 3
    ws = int(R.lib.ref_working_set_kb(n, n + k, 1))
    assert out.stdout.split() == ["band", "yes", "100", str(n + k), str((n + k) // n), str(ws)]


@pytest.mark.gpu
def test_matrix_market_symmetric_and_symmetrize(tmp_path):
    p = tmp_path / "sym.mtx"
    # symmetric file: lower triangle + diagonal stored, expanded on read
    write_mtx(p, 4, [0, 1, 2, 3, 1, 3], [0, 1, 2, 3, 0, 2], [4.0, 5.0, 6.0, 7.0, -1.0, 0.5], "symmetric")
    r = cli("verify", "--matrix", str(p), "--threads", "1,2")
    assert r.returncode == 0 and r.stdout.strip().endswith("VERIFY PASS"), r.stdout + r.stderr
    q = tmp_path / "asym.mtx"
    write_mtx(q, 3, [0, 1, 2, 2], [0, 1, 2, 0], [1.0, 2.0, 3.0, 4.0])
    r = cli("info", "--matrix", str(q))
    assert r.returncode == 1
    assert r.stderr.strip() == ("error: matrix 'asym' is structurally asymmetric (1 missing transposes, "
                                "0 missing diagonals); pass --symmetrize to pad with zeros")
    r = cli("verify", "--matrix", str(q), "--symmetrize", "--threads", "2")
    assert r.returncode == 0 and "VERIFY PASS" in r.stdout


@pytest.mark.gpu
def test_run_reports_reference_fields(tmp_path):
    out = tmp_path / "r.json"
    r = cli("run", "--gen", "random_sym:n=3000,density=0.003,seed=4", "--strategy", "buffers", "--accum", "interval",
            "--threads", "4", "--reps", "20", "--runs", "3", "--out", "json", str(out))
    assert r.returncode == 0, r.stderr
    head, row = r.stdout.strip().splitlines()
    assert head.split(",") == FIELDS
    vals = dict(zip(FIELDS, row.split(",")))
    assert vals["strategy"] == "buffers" and vals["accum"] == "interval" and vals["p"] == "4"
    assert vals["format"] == "csrc" and vals["reps"] == "20" and vals["runs"] == "3"
    j = json.loads(out.read_text())
    assert list(j.keys()) == FIELDS
    assert j["mflops_effective"] > 0 and j["median_total_seconds"] > 0
    assert math.isclose(j["mflops_effective"], 2 * j["nnz_full"] * j["reps"] / j["median_total_seconds"] / 1e6,
                        rel_tol=1e-9)
    for strat in ("seq", "colorful", "gather", "windowed", "atomic"):
        r = cli("run", "--gen", "band:n=5000,h=4", "--strategy", strat, "--threads", "4", "--reps", "10", "--runs", "1")
        assert r.returncode == 0, (strat, r.stderr)
        vals = dict(zip(FIELDS, r.stdout.strip().splitlines()[1].split(",")))
        assert vals["strategy"] == strat
        if strat == "colorful":
            assert int(vals["n_colors"]) >= 2
    r = cli("run", "--gen", "random_sym:n=3000,density=0.003,seed=4", "--format", "csr", "--reps", "20", "--runs", "1")
    assert r.returncode == 0, r.stderr
    vals = dict(zip(FIELDS, r.stdout.strip().splitlines()[1].split(",")))
    assert vals["format"] == "csr" and float(vals["mflops_true"]) > 0
    r = cli("run", "--config", "c2", "--strategy", "gather", "--reps", "50", "--runs", "3", "--out", "csv",
            str(tmp_path / "c2.csv"))
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "c2.csv").read_text().splitlines()[0].split(",") == FIELDS
