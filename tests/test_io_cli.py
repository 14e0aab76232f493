"""Reference text format (src/tridiagonal.cpp:60-91) and the SPEC bench CLI."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2605_26599_b200 as br
from paper_2605_26599_b200 import generators as G
from paper_2605_26599_b200.__main__ import accuracy, toeplitz_exact
from paper_2605_26599_b200.tridiag_io import read_tridiagonal, write_tridiagonal

ROOT = Path(__file__).resolve().parents[1]


def test_roundtrip_bitwise(tmp_path):
    d, e = G.generate("normal", 257)
    p = tmp_path / "t.txt"
    write_tridiagonal(br.TridiagonalMatrix(d, e), str(p))
    T = read_tridiagonal(str(p))
    assert np.array_equal(T.d, d) and np.array_equal(T.e, e)
    lines = p.read_text().split("\n")
    assert lines[0] == "257" and len([x for x in lines if x]) == 1 + 257 + 256


@pytest.mark.parametrize("text,msg", [("", "bad order line"), ("0\n", "bad order line"), ("x\n", "bad order line"),
                                      ("3\n1\n2\n", "missing diagonal entry"),
                                      ("3\n1\n2\n3\n0.5\n", "missing off-diagonal entry")])
def test_read_errors_mirror_reference(tmp_path, text, msg):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(br.InvalidArgument, match=msg):
        read_tridiagonal(str(p))


def test_read_missing_file():
    with pytest.raises(br.InvalidArgument, match="cannot open tridiagonal file"):
        read_tridiagonal("/nonexistent/t.txt")


def test_read_rejects_nonfinite(tmp_path):
    p = tmp_path / "nan.txt"
    p.write_text("2\n1\nnan\n0.5\n")
    with pytest.raises(br.InvalidArgument):
        read_tridiagonal(str(p))


def test_accuracy_examples():
    """SPEC.md:576-578."""
    lam = np.array([0.0, 0.5])
    assert accuracy(lam, lam, 0.5) == (0.0, 0.0)
    ef, eb = accuracy(np.array([0.0, 0.5 + 1e-10]), np.array([0.0, 0.5]), 0.5)
    assert ef == pytest.approx(1e-10) and eb == pytest.approx(1e-10)
    ef, _ = accuracy(np.array([100.0 + 1e-8]), np.array([100.0]), 1.0)
    assert ef == pytest.approx(1e-10)


def test_spec_families():
    """SPEC.md:567-569 examples: toeplitz n=3, clustered centre."""
    d, e = G.generate("toeplitz", 3)
    assert list(d) == [2, 2, 2] and list(e) == [0.25, 0.25]
    d, e = G.generate("clustered", 3)
    assert d[1] == 1.0 and e[0] == pytest.approx(1e-4 * (1 + 0.1 * np.cos(0.33)))
    assert np.allclose(toeplitz_exact(3, 2.0, 0.25), np.sort(np.linalg.eigvalsh(
        np.diag([2.0] * 3) + np.diag([0.25] * 2, 1) + np.diag([0.25] * 2, -1))))


def test_cli_refuses_cpu_solvers():
    r = subprocess.run([sys.executable, "-m", "paper_2605_26599_b200", "--solver", "qrql"], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 2 and "not part of this product" in r.stderr


@pytest.mark.gpu
def test_cli_records(tmp_path):
    p = tmp_path / "t.txt"
    d, e = G.generate("uniform", 3000)
    write_tridiagonal(br.TridiagonalMatrix(d, e), str(p))
    out = tmp_path / "lam.txt"
    r = subprocess.run([sys.executable, "-m", "paper_2605_26599_b200", "--family", "file", "--input", str(p),
                        "--out", str(out), "--trace-merges"], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout.strip().splitlines()[-1])
    assert rec["status"] == "ok" and rec["n"] == 3000 and rec["e_bwd"] <= 1e-12 and rec["trace"]
    lam = np.array([float(x) for x in out.read_text().split()])
    assert np.all(np.diff(lam) >= 0) and rec["checksum_sum"] == pytest.approx(float(np.sum(lam)))
    r = subprocess.run([sys.executable, "-m", "paper_2605_26599_b200", "--family", "toeplitz", "--n", "1024", "4096",
                        "--format", "csv"], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = r.stdout.strip().splitlines()
    assert rows[0].split(",")[:3] == ["family", "n", "solver"] and len(rows) == 3
    assert all(float(x.split(",")[5]) <= 1e-12 for x in rows[1:])  # e_fwd vs analytic


@pytest.mark.gpu
def test_cli_reduced_dense():
    r = subprocess.run([sys.executable, "-m", "paper_2605_26599_b200", "--family", "reduced", "--n", "500"],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rec = json.loads(r.stdout.strip().splitlines()[-1])
    assert rec["status"] == "ok" and rec["e_bwd"] <= 1e-12
