"""SPEC `cli` surface: FSK1 files, CSV clouds, solve / bench."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2602_03067_b200 import cli

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("dtype", ["double", "single"])
@pytest.mark.parametrize("labels", [False, True])
def test_fsk1_round_trip_bit_identical(tmp_path, dtype, labels):
    rng = np.random.default_rng(3)
    pts = rng.normal(size=(37, 5))
    lab = rng.integers(0, 9, size=37).astype(np.uint32) if labels else None
    p = tmp_path / "c.fsk"
    cli.write_point_cloud(p, pts, lab, dtype=dtype)
    got, glab = cli.read_point_cloud(p)
    want = pts if dtype == "double" else pts.astype(np.float32).astype(np.float64)
    assert np.array_equal(got, want)
    assert (glab is None) == (lab is None)
    if labels:
        assert np.array_equal(glab, lab)
    # write(read(x)) reproduces the file byte for byte
    q = tmp_path / "d.fsk"
    cli.write_point_cloud(q, got, glab, dtype=dtype)
    assert q.read_bytes() == p.read_bytes()


def test_fsk1_errors_name_the_problem(tmp_path):
    p = tmp_path / "c.fsk"
    cli.write_point_cloud(p, np.ones((4, 3)))
    raw = p.read_bytes()
    (tmp_path / "trunc.fsk").write_bytes(raw[:-8])
    with pytest.raises(cli.FormatError, match="expected 96"):
        cli.read_point_cloud(tmp_path / "trunc.fsk")
    (tmp_path / "magic.fsk").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(cli.FormatError, match="bad magic"):
        cli.read_point_cloud(tmp_path / "magic.fsk")
    (tmp_path / "short.fsk").write_bytes(raw[:10])
    with pytest.raises(cli.FormatError, match="truncated header"):
        cli.read_point_cloud(tmp_path / "short.fsk")


def test_csv_cloud_with_labels_round_trips_through_fsk1(tmp_path):
    c = tmp_path / "c.csv"
    c.write_text("x0,x1,label\n0.5,-1.25,3\n2,0,1\n")
    pts, lab = cli.read_csv_cloud(c)
    assert pts.shape == (2, 2) and list(lab) == [3, 1]
    cli.write_point_cloud(tmp_path / "c.fsk", pts, lab)
    p2, l2 = cli.read_point_cloud(tmp_path / "c.fsk")
    assert np.array_equal(p2, pts) and np.array_equal(l2, lab)


def test_uniform_weights_pass_naive_sum():
    for n in (1, 7, 100000):
        s = 0.0
        for v in cli.uniform(n):
            s += v
        assert abs(s - 1.0) <= 1e-12


@pytest.mark.gpu
def test_cli_solve_and_bench(tmp_path):
    env = dict(PYTHONPATH=str(ROOT))
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2602_03067_b200.cli", *a],
                                    capture_output=True, text=True, cwd=ROOT, timeout=600,
                                    env={**__import__("os").environ, **env})
    r = run("gen", str(tmp_path / "x.fsk"), "--n", "300", "--d", "3", "--seed", "1")
    assert r.returncode == 0, r.stderr
    r = run("gen", str(tmp_path / "y.fsk"), "--n", "250", "--d", "3", "--seed", "2")
    assert r.returncode == 0, r.stderr
    r = run("solve", str(tmp_path / "x.fsk"), str(tmp_path / "y.fsk"), "--eps", "0.5", "--iters",
            "20")
    assert r.returncode == 0, r.stderr
    vals = dict(line.split() for line in r.stdout.strip().splitlines())
    assert int(vals["iterations"]) == 20 and np.isfinite(float(vals["dual_cost"]))
    r = run("bench", "--n", "512", "--d", "3,64", "--iters", "5", "--deterministic")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "method,schedule,n,m,d,eps,iters,time_ms,peak_bytes,io_scalars,precision"
    assert len(lines) == 3
    # bad file -> exit code 1 (validation)
    (tmp_path / "bad.fsk").write_bytes(b"FSK1")
    r = run("solve", str(tmp_path / "bad.fsk"), str(tmp_path / "y.fsk"))
    assert r.returncode == 1
