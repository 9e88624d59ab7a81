"""The benchmark CLI (python -m paper_1709_00302_b200), modelled on the
reference's pkg/tests/test_cli.py: deterministic SplitMix64 inputs, the text
matrix format, the CSV schema, block sweeps, verification, dump/load and the
exit codes. Generator / format / config-error tests run on the CPU (the CLI
validates everything before touching the GPU); the rest are gpu tests."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1709_00302_b200 import (gen_general, gen_sym, load_matrix, save_matrix,
                                   sevp_nominal_flops, svd_nominal_flops)

HEADER = "algo,m,n,w,b,ts,tp,seconds,gflops,verify_max_dev,best"
G = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_1709_00302_b200", *args],
                          capture_output=True, text=True, timeout=600, cwd=ROOT)


def _rows(proc):
    lines = proc.stdout.strip().splitlines()
    assert lines and lines[0] == HEADER, proc.stderr
    return [line.split(",") for line in lines[1:]]


def _splitmix_ref(seed, i):
    """Independent big-int statement of the generator for one index."""
    mask = (1 << 64) - 1
    z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & mask
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
    z = z ^ (z >> 31)
    return float(z >> 11) * 2.0**-53 + 2.0**-54


# --- inputs (CPU) ---------------------------------------------------------------

def test_gen_matches_reference_golden():
    d = np.load(os.path.join(G, "cli.npz"))
    assert np.array_equal(gen_general(7, 5, 9), d["gen_general_7_5_9"])
    assert np.array_equal(gen_sym(6, 3), d["gen_sym_6_3"])
    assert np.array_equal(gen_general(33, 17, 123456789), d["gen_general_33_17_123456789"])


def test_gen_general_matches_stream():
    A = gen_general(5, 3, seed=42)
    for r in range(5):
        for c in range(3):
            assert A[r, c] == _splitmix_ref(42, c * 5 + r)  # column-major index
    big = gen_general(3, 2, (1 << 64) - 5)  # seed wraps mod 2^64
    assert big[2, 1] == _splitmix_ref((1 << 64) - 5, 5)


def test_gen_chunking_is_invisible():
    from paper_1709_00302_b200.cli import _splitmix64_unit

    a = _splitmix64_unit(1000, 11, chunk=7)
    assert np.array_equal(a, _splitmix64_unit(1000, 11))
    assert np.all((a > 0.0) & (a < 1.0))


def test_gen_sym_and_errors():
    S = gen_sym(64, 3)
    assert np.array_equal(S, S.T)
    G_ = gen_general(64, 64, 3)
    assert np.array_equal(S, (G_ + G_.T) / 2.0)
    with pytest.raises(ValueError):
        gen_general(0, 4, 0)


def test_matrix_text_format_matches_reference(tmp_path):
    ref = os.path.join(G, "matrix_4x3.txt")  # written by the reference's save_matrix
    A = load_matrix(ref)
    assert A.shape == (4, 3) and A[2, 0] == 1e-300 and np.signbit(A[1, 1])
    path = tmp_path / "m.txt"
    save_matrix(path, A)
    assert path.read_bytes() == open(ref, "rb").read()


def test_save_load_roundtrip_and_errors(tmp_path):
    A = gen_general(7, 5, 9) * 1e6 - 5e5
    path = tmp_path / "m.txt"
    save_matrix(path, A)
    assert np.array_equal(load_matrix(path), A)
    assert path.read_text().splitlines()[0] == "7 5"
    bad = tmp_path / "bad.txt"
    bad.write_text("2 2\n1.0\n2.0\n3.0\n")
    with pytest.raises(ValueError):
        load_matrix(bad)


def test_config_errors_exit_2(tmp_path):
    rect = tmp_path / "rect.txt"
    save_matrix(rect, gen_general(4, 5, 0))
    checks = [
        ("--algo", "sevp-v1", "--n", "24", "--w", "4", "--b", "3"),  # 2b > w
        ("--algo", "sevp-ref"),  # no --n and no --load
        ("--algo", "sevp-ref", "--n", "24", "--b", "40"),  # b > w
        ("--algo", "sevp-ref", "--n", "24", "--threads", "2", "--ts", "3"),
        ("--algo", "sevp-ref", "--n", "300", "--verify"),  # beyond oracle scale
        ("--algo", "svd-ref", "--n", "200", "--verify"),
        ("--algo", "nope", "--n", "8"),
        ("--algo", "sevp-ref", "--n", "24", "--b", "2", "--b-sweep"),
        ("--algo", "svd-triband", "--n", "24", "--w", "4", "--b", "2", "--b-sweep"),
        ("--algo", "sevp-ref", "--load", str(rect)),
        ("--algo", "sevp-ref", "--load", str(tmp_path / "missing.txt")),
        ("--algo", "depgraph", "--ratio", "2"),  # CPU analysis tool, not the GPU path
    ]
    for args in checks:
        proc = _run(*args)
        assert proc.returncode == 2, (args, proc.stderr)
        assert proc.stdout == "", args


# --- benchmark mode (GPU) -------------------------------------------------------

@pytest.mark.gpu
def test_basic_run_emits_one_csv_row():
    proc = _run("--algo", "sevp-ref", "--n", "24", "--w", "4", "--b", "2")
    assert proc.returncode == 0, proc.stderr
    rows = _rows(proc)
    assert len(rows) == 1
    algo, m, n, w, b, ts, tp, secs, gf, dev, best = rows[0]
    assert (algo, m, n, w, b) == ("sevp-ref", "24", "24", "4", "2")
    assert (ts, tp) == ("1", "0")
    assert float(secs) > 0.0 and dev == "" and best == ""
    assert float(gf) == sevp_nominal_flops(24) / float(secs) / 1e9


@pytest.mark.gpu
def test_gflops_column_is_nominal_over_seconds():
    proc = _run("--algo", "svd-ref", "--n", "20", "--m", "26", "--w", "4", "--b", "2")
    _, m, n, _, _, _, _, secs, gf, _, _ = _rows(proc)[0]
    assert float(gf) == svd_nominal_flops(26, 20) / float(secs) / 1e9


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["sevp-ref", "sevp-v1", "sevp-v2"])
def test_sevp_verify(algo):
    proc = _run("--algo", algo, "--n", "100", "--w", "8", "--b", "4", "--threads", "2",
                "--verify")
    assert proc.returncode == 0, proc.stderr
    dev = _rows(proc)[0][9]
    assert dev != "" and 0.0 <= float(dev) <= 1e-11 * 100


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["svd-triband", "svd-ref", "svd-sim", "svd-v1", "svd-v2"])
def test_svd_verify(algo):
    proc = _run("--algo", algo, "--n", "90", "--m", "120", "--w", "8", "--b", "4", "--verify")
    assert proc.returncode == 0, proc.stderr
    assert _rows(proc)[0][0] == algo


@pytest.mark.gpu
def test_wide_matrix_charges_the_transposed_problem():
    proc = _run("--algo", "svd-triband", "--m", "14", "--n", "20", "--w", "2", "--b", "2",
                "--verify")
    assert proc.returncode == 0, proc.stderr
    row = _rows(proc)[0]
    assert (row[1], row[2]) == ("14", "20")
    assert float(row[8]) == svd_nominal_flops(20, 14) / float(row[7]) / 1e9


@pytest.mark.gpu
def test_block_sweep_emits_best_row():
    proc = _run("--algo", "svd-ref", "--n", "20", "--m", "24", "--w", "4",
                "--b-sweep", "--b-start", "1", "--b-end", "4", "--b-step", "1")
    assert proc.returncode == 0, proc.stderr
    rows = _rows(proc)
    assert len(rows) == 5
    assert [r[4] for r in rows[:4]] == ["1", "2", "3", "4"]
    assert all(r[10] == "" for r in rows[:4])
    best = rows[4]
    assert best[10] == "1" and best[:10] in [r[:10] for r in rows[:4]]
    assert float(best[8]) == max(float(r[8]) for r in rows[:4])


@pytest.mark.gpu
def test_v1_sweep_defaults_cap_at_half_w():
    proc = _run("--algo", "sevp-v1", "--n", "30", "--w", "8", "--b-sweep", "--b-start", "2",
                "--b-step", "2")
    assert proc.returncode == 0, proc.stderr
    assert [r[4] for r in _rows(proc)[:-1]] == ["2", "4"]


@pytest.mark.gpu
def test_dump_and_load_reproduce_the_run(tmp_path):
    dump = tmp_path / "in.txt"
    p1 = _run("--algo", "sevp-ref", "--n", "20", "--w", "4", "--b", "2", "--seed", "5",
              "--dump", str(dump), "--verify")
    assert p1.returncode == 0, p1.stderr
    assert np.array_equal(load_matrix(dump), gen_sym(20, 5))
    p2 = _run("--algo", "sevp-ref", "--w", "4", "--b", "2", "--load", str(dump), "--verify")
    assert p2.returncode == 0, p2.stderr
    blank = lambda r: r[:7] + r[9:]  # noqa: E731  timing fields differ
    assert [blank(r) for r in _rows(p1)] == [blank(r) for r in _rows(p2)]


@pytest.mark.gpu
def test_trace_file_shows_lookahead_on_two_streams(tmp_path):
    trace = tmp_path / "trace.tsv"
    proc = _run("--algo", "sevp-v1", "--n", "300", "--w", "16", "--b", "8", "--threads", "2",
                "--trace", str(trace))
    assert proc.returncode == 0, proc.stderr
    recs = [line.split("\t") for line in trace.read_text().splitlines()]
    ids = [r[0] for r in recs]
    assert "qr@0" in ids and any(i.startswith("mid-head@") for i in ids)
    groups = {r[1] for r in recs}
    assert groups == {"seq", "par"}  # next panels on the panel stream
    for _, _, t0, t1 in recs:
        assert 0.0 <= float(t0) <= float(t1)
    # sequential schedule: no panel-stream records
    proc = _run("--algo", "sevp-v1", "--n", "300", "--w", "16", "--b", "8", "--threads", "2",
                "--ts", "0", "--trace", str(trace))
    assert proc.returncode == 0, proc.stderr
    assert {line.split("\t")[1] for line in trace.read_text().splitlines()} == {"par"}


@pytest.mark.gpu
def test_csv_is_stable_across_runs():
    args = ("--algo", "svd-v2", "--n", "24", "--w", "6", "--b", "4", "--threads", "2", "--verify")
    r1, r2 = _run(*args), _run(*args)
    assert r1.returncode == 0 and r2.returncode == 0
    blank = lambda r: r[:7] + r[9:]  # noqa: E731
    assert [blank(r) for r in _rows(r1)] == [blank(r) for r in _rows(r2)]
