"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the CPU oracle.  Needs a B200 (pytest -m gpu)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from tests.golden.cases import CASES, tet_hash  # noqa: E402


@pytest.fixture(scope="module")
def gq():
    from paper_1903_03406_b200 import _native
    _native.lib()
    return _native


def test_predicates_bit_exact(gq, golden_dir):
    g = np.load(os.path.join(golden_dir, "predicates.npz"))
    assert np.array_equal(gq.batch("orient3d", g["o3d_in"]), g["out_o3d"])
    assert np.array_equal(gq.batch("insphere", g["isp_in"]), g["out_isp"])
    assert np.array_equal(gq.batch("orient2d", g["o2d_in"]), g["out_o2d"])
    assert np.array_equal(gq.batch("incircle2d", g["icc_in"]), g["out_icc"])
    assert np.array_equal(gq.batch("incircle3d", g["inc3_in"]), g["out_inc3"])
    assert np.array_equal(gq.batch("encroaches_segment", g["eseg_in"]), g["out_eseg"])
    assert np.array_equal(gq.batch("encroaches_face", g["eface_in"]), g["out_eface"])
    cs = gq.batch("circumsphere_tet", g["o3d_in"][: len(g["out_csph"])])
    m = ~np.isnan(g["out_csph"])
    assert np.array_equal(np.isnan(cs), ~m)
    assert np.array_equal(cs[m], g["out_csph"][m])
    cc = gq.batch("circumcircle_tri", g["o3d_in"][: len(g["out_ccir"])][:, :9])
    m = ~np.isnan(g["out_ccir"])
    assert np.array_equal(cc[m], g["out_ccir"][m])


def test_predicates_random_vs_oracle(gq):
    import oracle
    rng = np.random.default_rng(7)
    for name, oname, w in (("orient3d", "or_orient3d", 12), ("insphere", "or_insphere", 15)):
        x = rng.uniform(-1, 1, (20000, w))
        # half of them snapped to a coarse grid: many exact zeros / ties
        x[::2] = np.round(x[::2] * 4) / 4
        assert np.array_equal(gq.batch(name, x), oracle.batch(oname, x))


@pytest.mark.parametrize("name", ["cube0", "cube100", "cube300", "c1", "seg1000", "rect600", "tri500", "oblique500"])
def test_refine_vs_reference(gq, golden_dir, name):
    from paper_1903_03406_b200 import RefineConfig, refine
    g = np.load(os.path.join(golden_dir, f"refine_{name}.npz"))
    build, B = CASES[name]
    mesh, rep = refine(build(), RefineConfig(B=float(g["B"])))
    steiner = int(g["steiner"])
    # north-star bar: Steiner count and residual bad tets within 2% of the reference
    assert abs(rep.steiner_points - steiner) <= max(1, 0.02 * steiner), (rep.steiner_points, steiner)
    assert abs(rep.bad_tet_count - int(g["bad_tet_count"])) <= max(2, 0.02 * int(g["bad_tet_count"]))
    mesh.audit()
    # conformity: every subsegment is an edge, every subface a face (audit), and
    # the subsegments of each input segment tile it
    if mesh.nv == len(g["points"]) and np.array_equal(mesh.points, g["points"]):
        # identical run: same tets too
        real = mesh.tv[(mesh.alive == 1) & (mesh.tv[:, 3] >= 0)]
        assert tet_hash(real) == str(g["tet_hash"])
