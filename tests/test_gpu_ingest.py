"""Device ingest of PCUT1B files (pcb_create_from_file) vs handles built from
host arrays: identical device state, identical solves."""
import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200 import io as pio
from paracut_b200.instances import make_instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wl,dims", [("cfg1", (40, 33)), ("cfg3", (30, 41)), ("cfg4", (12, 10, 14))])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_file_handle_equals_array_handle(tmp_path, wl, dims, precision):
    g = make_instance(wl, seed=3, dims=dims)
    p = tmp_path / "g.pcut"
    pio.write_grid(g, p)
    gf = pio.open_grid(p)
    A = _native.GridSolver(g, precision=precision)
    B = _native.GridSolver(gf, precision=precision)
    assert gf._grid is None  # the handle never built host arrays
    for S in (A, B):
        S.init_cold()
        S.run(12)
        S.shadow()
    assert np.array_equal(A.get_z(), B.get_z())
    ea, ga, da = A.check(np.array([0.0]))
    eb, gb, db = B.check(np.array([0.0]))
    assert np.array_equal(ea, eb) and np.array_equal(ga, gb) and da == db


def test_solve_from_file_matches_in_memory(tmp_path):
    g = make_instance("cfg2_int", seed=1, dims=(48, 40))
    p = tmp_path / "g.pcut"
    pio.write_grid(g, p)
    gf = pio.open_grid(p)
    cfg = pc.SolverConfig(gap_tol=1e-6, max_iters=3000, check_every=20)
    a = pc.solve(g, pc.decompose_grid(g), cfg)
    b = pc.solve(gf, pc.decompose_grid(gf), cfg)
    assert a.iterations == b.iterations and a.certified == b.certified
    assert np.array_equal(a.labeling, b.labeling) and a.energy == b.energy
    assert b.dual_state.fingerprint == pc.instance_fingerprint(g)
    assert gf._grid is None


def test_malformed_files_fail_in_the_library(tmp_path):
    g = make_instance("cfg1", seed=0, dims=(9, 8))
    p = tmp_path / "g.pcut"
    pio.write_grid(g, p)
    raw = p.read_bytes()
    bad = tmp_path / "bad.pcut"
    bad.write_bytes(raw[:-8])
    gf = pio.GridFile.__new__(pio.GridFile)  # bypass the Python-side size check
    gf.path, gf.dims, gf.connectivity = str(bad), g.dims, g.connectivity
    with pytest.raises(ValueError, match="truncated payload"):
        _native.GridSolver(gf, precision="f64")
    gf.path = str(tmp_path / "missing.pcut")
    with pytest.raises(ValueError, match="cannot open"):
        _native.GridSolver(gf, precision="f64")


def test_negative_edge_weight_in_file_is_rejected(tmp_path):
    """GridEnergy's 'edge weights must be nonnegative' (reference graph.py) on
    the device-ingest path, which never builds host arrays."""
    g = make_instance("cfg1", seed=0, dims=(9, 8))
    p = tmp_path / "g.pcut"
    pio.write_grid(g, p)
    raw = bytearray(p.read_bytes())
    off = 6 + 2 + 8 * 2 + 8 * g.n + 8 * 5  # sixth entry of the first direction array
    raw[off:off + 8] = np.array([-0.25], dtype="<f8").tobytes()
    bad = tmp_path / "neg.pcut"
    bad.write_bytes(bytes(raw))
    for precision in ("f64", "f32"):
        with pytest.raises(ValueError, match="nonnegative"):
            _native.GridSolver(pio.open_grid(bad), precision=precision)
