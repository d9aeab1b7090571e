"""The vectorised setup certifier (setup_fast.py) against the exact,
reference-order host path (plc.validate / hull_covered / facet_keep)."""

import numpy as np

from paper_1903_03406_b200 import PLC, synth
from paper_1903_03406_b200.plc import _exact_pair, _overlapping_pairs, hull_covered, validate
from paper_1903_03406_b200.prepare import facet_keep
from paper_1903_03406_b200 import setup_fast as sf


def _both(plc):
    return validate(plc, fast=True), validate(plc, fast=False)


def test_valid_inputs_agree():
    for plc in (synth.nested_surfaces(3000, level=2, torus=(24, 12)),
                synth.triangles_cloud(400, 30, 1),
                synth.config_plc("C2", scale=0.02),
                synth.config_plc("C1", scale=0.2)):
        f, e = _both(plc)
        assert f == e == []


def test_invalid_inputs_fall_back_to_the_exact_report():
    base = synth.nested_surfaces(500, level=1, torus=(12, 6))
    pts, segs, polys = list(base.points), list(base.segments), list(base.polygons)
    # a segment piercing the outer sphere
    a, b = len(pts), len(pts) + 1
    bad = PLC(points=pts + [(0.0, 0.0, 0.5), (0.0, 0.0, 1.5)], segments=segs + [(a, b)], polygons=polys)
    f, e = _both(bad)
    assert f == e and any(code == "segment-polygon-intersection" for code, _ in e)
    # crossing segments
    cross = PLC(points=[(0, 0, 0), (1, 1, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], segments=[(0, 1), (2, 3)])
    f, e = _both(cross)
    assert f == e == [("segment-segment-intersection", (0, 1))]
    # a triangle edge that is not a segment
    f, e = _both(PLC(points=pts, segments=segs[1:], polygons=polys))
    assert f == e and e[0][0] == "polygon-edge-not-in-segments"
    # duplicate point
    f, e = _both(PLC(points=pts + [pts[3]], segments=segs, polygons=polys))
    assert f == e and ("duplicate-point", (3, len(pts))) in e


def test_collinear_and_touching_segments():
    # collinear overlap, T-junction and a shared endpoint: exact decisions
    pts = [(0, 0, 0), (2, 0, 0), (1, 0, 0), (3, 0, 0), (1, -1, 0), (1, 1, 0), (0, 0, 1)]
    for segs in ([(0, 1), (2, 3)], [(0, 1), (2, 5)], [(0, 2), (2, 6)], [(0, 1), (4, 5)]):
        f, e = _both(PLC(points=pts, segments=segs))
        assert f == e


def test_overlapping_pairs_equals_the_sweep():
    rng = np.random.default_rng(5)
    lo = rng.uniform(0, 1, (3000, 3))
    hi = lo + rng.exponential(0.02, (3000, 3))
    hi[::97] += 0.5                                    # a few long boxes
    lo[5] = lo[6]; hi[5] = hi[6]                       # identical boxes
    got = {tuple(p) for p in sf.overlapping_pairs(lo, hi).tolist()}
    boxes = [(lo[k], hi[k]) for k in range(len(lo))]
    want = set(_overlapping_pairs(boxes))
    assert got == want


def test_exact_pair_matches_seg_poly_cases():
    base = synth.nested_surfaces(300, level=1, torus=(12, 6))
    nseg = len(base.segments)
    # every (segment, polygon) pair with a shared vertex is conflict-free
    for u in range(0, nseg, 7):
        i, j = base.segments[u]
        for pid, poly in enumerate(base.polygons):
            if i in poly or j in poly:
                assert not _exact_pair(base, u, nseg + pid)


def _keep_exact(plc, monkeypatch):
    monkeypatch.setattr(sf, "facet_axes", lambda q: np.full((len(q.polygons), 2), -1, dtype=np.int32))
    out = facet_keep(plc)
    monkeypatch.undo()
    return out


def test_facet_axes_and_hull(monkeypatch):
    plc = synth.nested_surfaces(2000, level=3, torus=(40, 20))
    fast = sf.facet_axes(plc)
    ok = fast[:, 0] >= 0
    assert ok.mean() > 0.9                       # ties (symmetric triangles) go to the exact path
    exact = _keep_exact(plc, monkeypatch)
    assert np.array_equal(fast[ok], exact[ok])
    assert np.array_equal(facet_keep(plc), exact)
    # nearly degenerate slivers go to the exact path (-1) or agree with it
    rng = np.random.default_rng(2)
    p = rng.uniform(-1, 1, (60, 3))
    p[1::3] = p[0::3] + 1e-12 * rng.uniform(-1, 1, (20, 3))
    q = PLC(points=[tuple(x) for x in p], segments=[], polygons=[(3 * k, 3 * k + 1, 3 * k + 2) for k in range(20)])
    fa = sf.facet_axes(q)
    ex = _keep_exact(q, monkeypatch)
    ok = fa[:, 0] >= 0
    assert np.array_equal(fa[ok], ex[ok])
    # hull coverage: the certifier only ever confirms what the exact test says
    tet = PLC(points=[(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (0.1, 0.1, 0.1)],
              segments=[(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)],
              polygons=[(0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)])
    for plc in (tet, synth.nested_surfaces(100, level=2, torus=(12, 6))):
        got = hull_covered(plc)
        monkeypatch.setattr(sf, "certify_hull_covered", lambda q, h: None)
        assert got == hull_covered(plc)
        monkeypatch.undo()
    assert hull_covered(tet)
