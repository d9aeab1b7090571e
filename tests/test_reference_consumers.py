"""Drop-in check of the exported Mesh: the reference's own consumers
(tetrefine.stats.analyze, stats.py:88-99; tetrefine.formats.write_mesh,
formats.py:245-263) read it and produce exactly what this package's
implementations produce.  The reference is importable only in the build
container (/root/reference); elsewhere the test is skipped."""

import os
import sys

import numpy as np
import pytest

import oracle  # test infrastructure
from paper_1903_03406_b200 import formats, stats, synth
from paper_1903_03406_b200.mesh import Mesh, bbox_diag_of

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")


@pytest.fixture(scope="module")
def tetrefine():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    import tetrefine.formats
    import tetrefine.stats
    return tetrefine


@pytest.fixture(scope="module")
def mesh():
    plc = synth.segments_cloud(400, 6, 1)
    o = oracle.refine(plc, B=1.6)
    arrays = {k: o[k] for k in ("points", "vert_origin", "vert_tet", "tv", "tn", "alive", "sub_mask", "seg_mask",
                                "ratio", "skip_flag")}
    segs = {(int(u), int(v)): int(s) for u, v, s in o["subsegments"]}
    faces = {(int(a), int(b), int(c)): int(p) for a, b, c, p in o["subfaces"]}
    return Mesh(arrays, segs, faces, bbox_diag_of(o["points"]))


def test_reference_stats_analyze_reads_the_mesh(tetrefine, mesh):
    ref = tetrefine.stats.analyze(mesh, 1.6)
    own = stats.analyze(mesh, 1.6)
    assert ref.input_points == own.input_points and ref.steiner_points == own.steiner_points
    assert ref.tet_count == own.tet_count and ref.bad_tet_count == own.bad_tet_count
    assert list(ref.dihedral_histogram) == list(own.dihedral_histogram)


def test_reference_write_mesh_reads_the_mesh(tetrefine, mesh, tmp_path):
    a = [tmp_path / f"ref.{e}" for e in ("node", "ele", "face")]
    b = [tmp_path / f"own.{e}" for e in ("node", "ele", "face")]
    tetrefine.formats.write_mesh(mesh, *map(str, a))
    formats.write_mesh(mesh, *map(str, b))
    for x, y in zip(a, b):
        assert x.read_bytes() == y.read_bytes(), x.name
