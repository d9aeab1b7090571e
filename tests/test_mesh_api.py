"""The exported Mesh's query API (tetrefine.mesh.Mesh, mesh.py:236-391):
adjacency queries and point location, checked against brute force on a mesh
the CPU oracle built (the oracle is pinned bit-identical to the reference)."""

import numpy as np
import pytest

import oracle  # test infrastructure
from paper_1903_03406_b200 import exactnp, synth
from paper_1903_03406_b200.mesh import GHOST, OUTSIDE, Mesh, bbox_diag_of


@pytest.fixture(scope="module")
def mesh():
    plc = synth.cube_points(60, 3)
    o = oracle.refine(plc, B=2.0)
    arrays = {k: o[k] for k in ("points", "vert_origin", "vert_tet", "tv", "tn", "alive", "sub_mask", "seg_mask",
                                "ratio", "skip_flag")}
    segs = {(int(u), int(v)): int(s) for u, v, s in o["subsegments"]}
    faces = {(int(a), int(b), int(c)): int(p) for a, b, c, p in o["subfaces"]}
    return Mesh(arrays, segs, faces, bbox_diag_of(o["points"]))


def test_tets_around_vertex_and_edges(mesh):
    A = np.flatnonzero(mesh.alive == 1)
    rng = np.random.default_rng(0)
    for v in rng.choice(mesh.nv, 25, replace=False):
        brute = {int(t) for t in A if v in mesh.tv[t]}
        assert set(mesh.tets_around_vertex(int(v))) == brute
    for (u, v) in list(mesh.subsegments)[:20]:
        assert mesh.edge_exists(u, v)
        ring = mesh.edge_link_vertices(u, v)
        brute = {int(w) for t in A if u in mesh.tv[t] and v in mesh.tv[t] for w in mesh.tv[t]} - {u, v, GHOST}
        assert ring == brute
    assert not mesh.edge_exists(0, 10 ** 9)


def test_find_tet_with_face(mesh):
    for key in list(mesh.subfaces)[:30]:
        t, i = mesh.find_tet_with_face(key)
        assert t >= 0 and mesh.face_key(t, i) == key
        u, j = mesh.neighbor(t, i)
        assert mesh.face_key(u, j) == key
    assert mesh.find_tet_with_face((0, 1, 10 ** 9)) == (-1, -1)


def test_locate(mesh):
    rng = np.random.default_rng(1)
    real = np.array(mesh.real_tets())
    q = mesh.tv[real]
    P = mesh.points
    for p in rng.uniform(0.0, 1.0, (30, 3)):
        ref = mesh.locate(p)
        assert ref.kind == "tet"
        # brute force: lowest real tet with p inside or on the boundary
        inside = np.ones(len(real), dtype=bool)
        for f in ((1, 2, 3), (0, 3, 2), (0, 1, 3), (0, 2, 1)):
            s = exactnp.orient3d_batch(P[q[:, f[0]]], P[q[:, f[1]]], P[q[:, f[2]]], np.repeat(p[None], len(real), 0))
            inside &= s <= 0
        assert ref.index == int(real[inside].min())
    # a mesh vertex: the lowest incident real tet
    v = int(mesh.tv[real[5], 2])
    assert mesh.locate(P[v]).index == min(t for t in real if v in mesh.tv[t])
    assert mesh.locate((5.0, 5.0, 5.0)) == OUTSIDE
