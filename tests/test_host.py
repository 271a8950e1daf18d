"""Host-side logic without a GPU: data model, decomposition, config, generator,
bench helpers, and the C-ABI library's exported surface."""
import os
import re

import numpy as np
import pytest

import paracut_b200 as pc
from paracut_b200 import _native
from paracut_b200.instances import CONFIGS, algorithmic_bytes, make_instance
from conftest import ROOT, aar_cases, golden_grid


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "paracut_b200.h")).read()
    decl = set(re.findall(r"\b(pcb_[A-Za-z_0-9]+)\s*\(", hdr))
    assert decl, "no declarations parsed"
    L = _native.lib()
    missing = [s for s in decl if not hasattr(L, s)]
    assert not missing, missing
    assert decl == set(_native.EXPORTS)
    assert L.pcb_version() >= 1


def test_no_device_raises_runtime_error_not_fallback():
    # on this CPU-only container every device entry point must fail loudly
    try:
        n = _native.device_count()
    except RuntimeError:
        return
    if n == 0:
        pytest.skip("device count 0 without error")


@pytest.mark.parametrize("name", aar_cases() + ["cfg1.npz", "kat.npz"])
def test_fingerprint_matches_reference(name):
    g, d = golden_grid(name)
    gg = pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)
    assert pc.instance_fingerprint(gg) == str(d["fingerprint"])


@pytest.mark.parametrize("name", aar_cases())
def test_materialised_classes_match_oracle_csr(name):
    from oracle import oracle as orc
    g, _ = golden_grid(name)
    gg = pc.GridEnergy(g.dims, g.connectivity, g.w, g.dir_weights)
    dec = pc.decompose_grid(gg)
    ours = dec.classes
    ref = orc.decompose(g)
    assert len(ours) == len(ref) == dec.r
    for a, b in zip(ours, ref):
        assert np.array_equal(a.node_idx, b.node_idx)
        assert np.array_equal(a.chain_ptr, b.chain_ptr)
        assert np.array_equal(a.edge_w, b.edge_w)
    assert np.all(dec.degree == dec.r)
    assert dec.tv(np.arange(g.n, dtype=float)) == pytest.approx(
        sum(c.tv(np.arange(g.n, dtype=float)) for c in ours))


def test_grid_energy_validation_and_energy():
    with pytest.raises(ValueError):
        pc.GridEnergy((3, 3), "2D-5", np.zeros(9), [])
    with pytest.raises(ValueError):
        pc.GridEnergy((3, 3), "3D-6", np.zeros(9), [])
    with pytest.raises(ValueError):
        pc.GridEnergy((3, 3), "2D-4", np.zeros(8), [np.ones((3, 2)), np.ones((2, 3))])
    with pytest.raises(ValueError):
        pc.GridEnergy((3, 3), "2D-4", np.zeros(9), [np.ones((3, 2)), np.ones((3, 3))])
    with pytest.raises(ValueError):
        pc.GridEnergy((3, 3), "2D-4", np.zeros(9), [-np.ones((3, 2)), np.ones((2, 3))])
    g = pc.GridEnergy((2, 2), "2D-4", np.array([1.0, -1.0, 0.5, 0.0]),
                      [np.array([[2.0], [0.0]]), np.array([[1.0, 3.0]])])
    x = np.array([1, 0, 0, 0])
    assert g.energy(x) == pytest.approx(2.0 + 1.0 - 1.0)
    assert g.num_edges == 3
    ei, ej, ea = g.edge_arrays()
    assert list(zip(ei, ej, ea)) == [(0, 1, 2.0), (0, 2, 1.0), (1, 3, 3.0)]
    h = g.scaled_pairwise(0.5)
    assert h.dir_weights[0][0, 0] == 1.0
    with pytest.raises(ValueError):
        g.scaled_pairwise(-1)


def test_solver_config_validation():
    with pytest.raises(ValueError, match="algorithm"):
        pc.SolverConfig(algorithm="newton")
    with pytest.raises(ValueError, match="max_iters"):
        pc.SolverConfig(max_iters=0)
    with pytest.raises(ValueError, match="tolerances"):
        pc.SolverConfig(dual_tol=-1)
    with pytest.raises(ValueError, match=">= 1"):
        pc.SolverConfig(check_every=0)
    with pytest.raises(ValueError, match="precision"):
        pc.SolverConfig(precision="f16")
    with pytest.raises(ValueError, match="thresholds"):
        pc.SolverConfig(thresholds=tuple(range(9)))
    with pytest.raises(ValueError, match="polish"):
        pc.SolverConfig(polish_stall=-1)
    assert pc.SolverConfig().thresholds == (0.0,)


def test_threshold_and_level_sets():
    x = np.array([-1.0, 0.0, 1e-300, 2.0])
    assert pc.threshold(x).tolist() == [0, 0, 1, 1]
    ls = pc.level_sets(np.array([0.5, -0.2, 0.5, 0.0]))
    assert len(ls) == 4 and ls[0].tolist() == [1, 1, 1, 1] and ls[-1].tolist() == [0] * 4


def test_jaccard_packed_equals_unpacked():
    from paracut_b200.certify import jaccard_packed
    rng = np.random.default_rng(0)
    from paracut_b200 import _native
    for n in (1, 7, 8, 9, 63, 64, 65, 1000, 100003):
        a = (rng.random(n) < 0.4).astype(np.uint8)
        b = (rng.random(n) < 0.6).astype(np.uint8)
        ref = pc.jaccard_distance(a, b)
        assert jaccard_packed(np.packbits(a), np.packbits(b)) == ref
        assert _native.jaccard_packed(np.packbits(a), np.packbits(b)) == ref  # host popcount
    z = np.zeros(5, np.uint8)
    assert _native.jaccard_packed(z, z) == 0.0 == pc.jaccard_distance(z, z)


def test_generator_reproduces_cfg1_fixture():
    # pins the synthetic generator: cfg1 seed 0 must be byte-identical to the
    # instance the golden reference run used
    g, d = golden_grid("cfg1.npz")
    ours = make_instance("cfg1", seed=0)
    assert np.array_equal(ours.w, d["w"])
    for k, a in enumerate(ours.dir_weights):
        assert np.array_equal(a, d["dw%d" % k])


def test_integer_variant_properties():
    g = make_instance(CONFIGS["cfg2_int"], seed=0, dims=(128, 128))
    assert np.all(g.w == np.rint(g.w)) and g.w.min() >= -10 and g.w.max() <= 10
    for a in g.dir_weights:
        assert np.all(a == np.rint(a)) and a.min() >= 0 and a.max() <= 5
    zero = sum(int((a == 0).sum()) for a in g.dir_weights) / sum(a.size for a in g.dir_weights)
    assert 0.05 < zero < 0.6


def test_algorithmic_bytes_match_baseline_table():
    # cfg1 fp64 3.67 MB, cfg3 fp32 872.3 MB, cfg4 fp32 670.3 MB
    def fake(dims, conn):
        from paracut_b200.graph import DIRECTIONS, direction_shape
        n = int(np.prod(dims))
        return pc.GridEnergy(dims, conn, np.zeros(n),
                             [np.ones(direction_shape(dims, d)) for d in DIRECTIONS[conn]])
    assert algorithmic_bytes(fake((256, 256), "2D-4"), 2, 8) / 1e6 == pytest.approx(3.67, abs=0.01)
    assert algorithmic_bytes(fake((4096, 4096), "2D-8"), 4, 4) / 1e6 == pytest.approx(872.3, abs=0.1)
    assert algorithmic_bytes(fake((256, 256, 256), "3D-6"), 3, 4) / 1e6 == pytest.approx(670.3, abs=0.1)


def test_bench_helpers():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    g = make_instance("cfg4", seed=0, dims=(40, 30, 20))
    g8 = make_instance("cfg3", seed=0, dims=(20, 30))
    fe = bench._family_edges(g8)
    assert sum(fe) == sum(int(np.count_nonzero(a)) for a in g8.dir_weights)
    # the CPU leg runs on the whole instance at all cores and one core
    cb = bench.cpu_baseline(make_instance("cfg4", seed=0, dims=(8, 16, 16)), "cfg4", 2, 1,
                            ttc_iters=100)
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["one_core"]["cores"] == 1
    assert "8x16x16" in cb["sample"] and cb["time_to_cut"]["extrapolated"]
    assert cb["time_to_cut"]["value"] == pytest.approx(cb["s_per_iter"] * 100)


def test_rank_parts_equal_the_sliced_instance():
    """A sharded rank's slab and pencil from the box generator (make_part, the
    host reference of pcb_create_synthetic_box) equal the slices of the whole
    instance that SlabGeometry takes."""
    from paracut_b200.distributed import SlabGeometry
    from paracut_b200.instances import make_part
    for name, dims, P in (("cfg4", (8, 12, 16), 4), ("cfg2", (16, 24), 4), ("cfg5_int", (4, 8, 8), 2)):
        g = make_instance(name, seed=3, dims=dims)
        geo = SlabGeometry(dims, CONFIGS[name].connectivity, P)
        for rk in range(P):
            for desc, ref in zip(geo.parts(rk), (geo.slab_grid(g, rk), geo.pencil_grid(g, rk))):
                o, e, d, m = desc
                part = make_part(name, 3, dims, o, e, d, m)
                assert part.dims == ref.dims and np.array_equal(part.w, ref.w)
                for x, y in zip(part.dir_weights, ref.dir_weights):
                    assert x.shape == y.shape and np.array_equal(x, y)
