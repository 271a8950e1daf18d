"""Command line front end (paracut_b200.cli) -- reference pkg/tests/test_cli.py
cases; the ones that solve need the GPU."""
import os

import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import cli
from paracut_b200 import io as pio
from paracut_b200.graph import DIRECTIONS, direction_shape


def _tiny_grid(rng, conn, dims):
    w = rng.uniform(-3, 3, int(np.prod(dims)))
    dws = [rng.uniform(0, 2, direction_shape(dims, d))
           * (rng.uniform(size=direction_shape(dims, d)) < 0.8) for d in DIRECTIONS[conn]]
    return pc.GridEnergy(dims, conn, w, dws)


@pytest.fixture
def grid_file(tmp_path):
    g = _tiny_grid(np.random.default_rng(7), "2D-8", (9, 11))
    p = tmp_path / "g.pcut"
    pio.write_grid(g, p)
    return str(p)


@pytest.fixture
def dimacs_file(tmp_path):
    p = tmp_path / "c.max"  # a general instance in DIMACS max-flow form
    p.write_text("p max 5 4\nn 4 s\nn 5 t\na 4 1 1.0\na 2 5 2.0\na 1 2 0.5\na 2 1 0.5\n")
    return str(p)


def test_usage_and_io_errors_without_a_device(tmp_path, grid_file, dimacs_file, capsys):
    assert cli.main(["solve", "--input", grid_file, "--algo", "maxflow"]) == cli.EXIT_USAGE
    assert cli.main(["solve", "--input", dimacs_file]) == cli.EXIT_USAGE
    assert "general instance" in capsys.readouterr().err
    assert cli.main(["solve", "--input", str(tmp_path / "missing")]) == cli.EXIT_IO
    bad = tmp_path / "bad"
    bad.write_bytes(b"PCUT1B\x09\x02")
    assert cli.main(["solve", "--input", str(bad)]) == cli.EXIT_IO
    assert cli.main(["solve", "--input", grid_file, "--scale-pairwise", "-1"]) == cli.EXIT_USAGE
    assert cli.main(["solve", "--input", dimacs_file, "--format", "grid"]) == cli.EXIT_IO
    with pytest.raises(SystemExit):
        cli.main(["solve"])  # argparse: --input required


def test_threads_default_from_environment(monkeypatch):
    monkeypatch.setenv("PARACUT_THREADS", "6")
    assert cli._default_threads() == 6
    monkeypatch.setenv("PARACUT_THREADS", "x")
    assert cli._default_threads() == 1


@pytest.mark.gpu
def test_solve_writes_labeling_and_artifacts(grid_file, tmp_path, capsys):
    out, tr, dual = tmp_path / "lab.txt", tmp_path / "t.csv", tmp_path / "s.dual"
    rc = cli.main(["solve", "--input", grid_file, "--gap-tol", "1e-6", "--out", str(out),
                   "--trace", str(tr), "--save-dual", str(dual)])
    text = capsys.readouterr().out
    assert rc == cli.EXIT_OK
    lines = dict(l.split(" ", 1) for l in text.strip().splitlines())
    lab = np.array([int(v) for v in out.read_text().split()], dtype=np.uint8)
    g = pio.read_grid(grid_file)
    assert float(lines["energy"]) == pytest.approx(g.energy(lab), abs=1e-9)
    assert float(lines["gap"]) <= 1e-6
    assert tr.read_text().splitlines()[0] == "iter,gap,dual_objective,jaccard_to_final,wall_ms"
    st = pio.load_dual(dual)
    assert st.fingerprint == pc.instance_fingerprint(g)
    # same answer as the in-memory API (device ingest changes nothing)
    res = pc.solve(g, pc.decompose_grid(g), pc.SolverConfig(gap_tol=1e-6))
    assert np.array_equal(res.labeling, lab)
    assert np.array_equal(res.dual_state.y, st.y) and np.array_equal(res.dual_state.z, st.z)


@pytest.mark.gpu
def test_solve_warm_start_and_fingerprint_guard(grid_file, tmp_path, capsys):
    dual = tmp_path / "s.dual"
    assert cli.main(["solve", "--input", grid_file, "--max-iters", "30", "--save-dual",
                     str(dual)]) in (cli.EXIT_OK, cli.EXIT_NOT_CERTIFIED)
    capsys.readouterr()
    assert cli.main(["solve", "--input", grid_file, "--warm-start", str(dual),
                     "--gap-tol", "1e-6"]) == cli.EXIT_OK
    other = tmp_path / "o.pcut"
    pio.write_grid(_tiny_grid(np.random.default_rng(8), "2D-8", (9, 11)), other)
    assert cli.main(["solve", "--input", str(other), "--warm-start", str(dual)]) == cli.EXIT_IO
    assert "fingerprint" in capsys.readouterr().err
    assert cli.main(["solve", "--input", str(other), "--warm-start", str(dual), "--force",
                     "--max-iters", "5"]) in (cli.EXIT_OK, cli.EXIT_NOT_CERTIFIED)


@pytest.mark.gpu
def test_solve_uncertified_exit_and_algorithms(grid_file, capsys):
    assert cli.main(["solve", "--input", grid_file, "--max-iters", "1", "--check-every",
                     "1"]) == cli.EXIT_NOT_CERTIFIED
    for algo in ("bcd", "ap", "fista"):
        assert cli.main(["solve", "--input", grid_file, "--algo", algo, "--gap-tol",
                         "1e-6"]) == cli.EXIT_OK
    assert cli.main(["solve", "--input", grid_file, "--precision", "f32", "--polish-iters",
                     "200", "--gap-tol", "1e-6", "--level-sets"]) == cli.EXIT_OK
