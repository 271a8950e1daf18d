"""Row families fed by TMA (the drift box transposed in to_z, node-order
outputs as per-lane vectors) against the per-lane cp.async sweep: the same
arithmetic in the same order, so states, step norms and shadows are bitwise
equal.  PCB_ROW_TMA=0 (read when a handle builds its tensor maps) selects the
cp.async path for the reference run."""
import os

import numpy as np
import pytest

from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, make_instance

pytestmark = pytest.mark.gpu


def _run(g, precision, iters, row_tma):
    old = os.environ.get("PCB_ROW_TMA")
    os.environ["PCB_ROW_TMA"] = "1" if row_tma else "0"
    try:
        S = _native.GridSolver(g, precision=precision)
    finally:
        if old is None:
            del os.environ["PCB_ROW_TMA"]
        else:
            os.environ["PCB_ROW_TMA"] = old
    try:
        S.init_cold()
        norms = S.run(iters)
        S.shadow()
        y = S.shadow_get()
        z = S.get_z()
        return np.asarray(norms), np.array(z, copy=True), np.array(y, copy=True)
    finally:
        S.close()


@pytest.mark.parametrize("spec,dims,prec,iters", [
    ("cfg2", (96, 128), "f32", 60),      # 2D-4 rows (split into merge-point units)
    ("cfg4", (24, 20, 64), "f32", 60),   # 3D x lines
    ("cfg3", (64, 96), "f32", 40),       # 2D-8: rows on TMA, zig-zags on cp.async
    ("cfg4", (16, 32, 48), "f64s", 40),  # fp64 split mode
    ("cfg2", (64, 1024), "f32", 30),     # long rows
])
def test_row_tma_bitwise(spec, dims, prec, iters):
    g = make_instance(CONFIGS[spec], seed=3, dims=dims)
    n1, z1, y1 = _run(g, prec, iters, True)
    n0, z0, y0 = _run(g, prec, iters, False)
    assert np.array_equal(z1, z0)
    assert np.array_equal(y1, y0)
    assert np.array_equal(n1, n0)


def test_row_tma_odd_rows_fall_back():
    # rows whose length is not a multiple of 4 keep the cp.async sweep
    g = make_instance(CONFIGS["cfg2"], seed=4, dims=(40, 54))
    n1, z1, _ = _run(g, "f32", 20, True)
    n0, z0, _ = _run(g, "f32", 20, False)
    assert np.array_equal(z1, z0)
