"""Piecewise linear complex input type, exact validation and domain closure.

Host-side setup of ``refine()``; the behaviour follows
/root/reference/pkg/src/tetrefine/plc.py (PLC :19-32, validate :267-383,
unit_cube :386-408) and the domain closure of refine.py:421-506
(``_hull_covered`` / ``augment_with_box``).  Every geometric decision is made
in exact rational arithmetic (``fractions.Fraction`` over the raw doubles),
so validation never flips on near-degenerate input.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .errors import EmptyPLC


@dataclass
class PLC:
    """Points P, segments E (index pairs) and polygons F (index cycles whose
    boundary edges are members of E).  Normalised like plc.py:29-32."""

    points: list = field(default_factory=list)
    segments: list = field(default_factory=list)
    polygons: list = field(default_factory=list)

    def __post_init__(self):
        self.points = [tuple(float(c) for c in p) for p in self.points]
        self.segments = [tuple(int(i) for i in s) for s in self.segments]
        self.polygons = [tuple(int(i) for i in poly) for poly in self.polygons]

    @classmethod
    def _normalised(cls, points, segments, polygons):
        """Build from lists that are already in normal form (no re-conversion)."""
        obj = cls.__new__(cls)
        obj.points, obj.segments, obj.polygons = points, segments, polygons
        return obj


def points_array(plc: PLC) -> np.ndarray:
    """(n, 3) float64 view of plc.points, converted once per PLC object (the
    list is the public, reference-compatible representation)."""
    cache = plc.__dict__.get("_points_np")
    if cache is None or cache[0] is not plc.points or len(cache[1]) != len(plc.points):
        arr = np.asarray(plc.points, dtype=np.float64).reshape(-1, 3)
        plc.__dict__["_points_np"] = cache = (plc.points, arr)
    return cache[1]


def polygon_index_array(plc: PLC) -> np.ndarray:
    """All polygon vertex indices, flattened (one conversion of the list)."""
    polys = plc.polygons
    try:
        return np.asarray(polys, dtype=np.int64).reshape(-1)     # uniform polygons (all triangles, ...)
    except ValueError:
        return np.fromiter((v for p in polys for v in p), dtype=np.int64)


def bounding_box(plc: PLC):
    if not plc.points:
        raise EmptyPLC("PLC has no points")
    arr = points_array(plc)
    return tuple(float(x) for x in arr.min(axis=0)), tuple(float(x) for x in arr.max(axis=0))


def bbox_diagonal(plc: PLC) -> float:
    lo, hi = bounding_box(plc)
    return math.dist(lo, hi)


# ---------------------------------------------------------------------------
# exact primitives on Fractions

def _F(p):
    return tuple(Fraction(c) for c in p)


def _sign(x):
    return (x > 0) - (x < 0)


def _o2(a, b, c):
    return _sign((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]))


def _o3(a, b, c, d):
    u = [b[k] - a[k] for k in range(3)]
    v = [c[k] - a[k] for k in range(3)]
    w = [d[k] - a[k] for k in range(3)]
    return _sign(u[0] * (v[1] * w[2] - v[2] * w[1]) - u[1] * (v[0] * w[2] - v[2] * w[0])
                 + u[2] * (v[0] * w[1] - v[1] * w[0]))


def _cross(u, v):
    return (u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0])


def _collinear(a, b, c):
    return _cross([b[k] - a[k] for k in range(3)], [c[k] - a[k] for k in range(3)]) == (0, 0, 0)


def _proj_axis(pts):
    """Axis of the largest |component| of the exact fan normal (first on
    ties), plc.py:73-85."""
    f = [_F(p) for p in pts]
    n = [Fraction(0)] * 3
    for i in range(1, len(f) - 1):
        c = _cross([f[i][k] - f[0][k] for k in range(3)], [f[i + 1][k] - f[0][k] for k in range(3)])
        n = [n[k] + c[k] for k in range(3)]
    mags = [abs(x) for x in n]
    best = 0
    for k in (1, 2):
        if mags[k] > mags[best]:
            best = k
    return best


def _drop(p, axis):
    return tuple(p[k] for k in range(3) if k != axis)


def _between(a, b, p):
    """p strictly inside segment ab (collinear inputs, any dimension)."""
    dot = sum((p[k] - a[k]) * (b[k] - a[k]) for k in range(len(a)))
    lsq = sum((b[k] - a[k]) ** 2 for k in range(len(a)))
    return 0 < dot < lsq


def point_in_polygon_2d(poly, q):
    """q inside or on the boundary of simple polygon poly (exact)."""
    poly = [tuple(Fraction(c) for c in p) for p in poly]
    q = tuple(Fraction(c) for c in q)
    n = len(poly)
    for i in range(n):
        a, b = poly[i], poly[(i + 1) % n]
        if _o2(a, b, q) == 0 and (q == a or q == b or _between(a, b, q)):
            return True
    inside = False
    for i in range(n):
        (ax, ay), (bx, by) = poly[i], poly[(i + 1) % n]
        if (ay > q[1]) != (by > q[1]):
            if ax + (q[1] - ay) * (bx - ax) / (by - ay) > q[0]:
                inside = not inside
    return inside


def _segs_touch_2d(a, b, c, d, shared):
    o1, o2, o3, o4 = _o2(a, b, c), _o2(a, b, d), _o2(c, d, a), _o2(c, d, b)
    if shared:
        return ((o1 == 0 and _between(a, b, c)) or (o2 == 0 and _between(a, b, d))
                or (o3 == 0 and _between(c, d, a)) or (o4 == 0 and _between(c, d, b)))
    if o1 == 0 and o2 == 0:
        return (_between(a, b, c) or _between(a, b, d) or _between(c, d, a) or _between(c, d, b)
                or a in (c, d) or b in (c, d))
    return o1 * o2 <= 0 and o3 * o4 <= 0


def _segs_conflict(a, b, c, d):
    """Open parts of segments ab, cd meet (anything but a shared endpoint)."""
    a, b, c, d = _F(a), _F(b), _F(c), _F(d)
    shared = {a, b} & {c, d}
    if len(shared) == 2:
        return True
    if _o3(a, b, c, d) != 0:
        return False
    if not (_collinear(a, b, c) and _collinear(a, b, d)):
        for axis in range(3):
            a2, b2, c2, d2 = (_drop(p, axis) for p in (a, b, c, d))
            if (_o2(a2, b2, c2), _o2(a2, b2, d2), _o2(c2, d2, a2), _o2(c2, d2, b2)) == (0, 0, 0, 0):
                continue
            return _segs_touch_2d(a2, b2, c2, d2, shared)
        return False
    for p, q in ((c, d), (d, c)):
        if p in shared:
            other = b if p == a else a
            return _between(a, b, q) or _between(p, q, other)
    return _between(a, b, c) or _between(a, b, d) or _between(c, d, a) or _between(c, d, b)


def _seg_poly_conflict(points, seg, poly):
    i, j = seg
    n = len(poly)
    if i in poly and j in poly:
        k = poly.index(i)
        if poly[(k + 1) % n] == j or poly[(k - 1) % n] == j:
            return False
    a, b = _F(points[i]), _F(points[j])
    verts = [_F(points[v]) for v in poly]
    p0, p1, p2 = verts[0], verts[1], verts[2]
    if _collinear(p0, p1, p2):
        for v in verts[3:]:
            if not _collinear(p0, p1, v):
                p2 = v
                break
    sa, sb = _o3(p0, p1, p2, a), _o3(p0, p1, p2, b)
    if sa * sb > 0:
        return False
    axis = _proj_axis([points[v] for v in poly])
    v2 = [_drop(v, axis) for v in verts]
    if sa == 0 and sb == 0:
        a2, b2 = _drop(a, axis), _drop(b, axis)
        if point_in_polygon_2d(v2, tuple((a2[k] + b2[k]) / 2 for k in range(2))):
            return True
        return any(idx not in poly and point_in_polygon_2d(v2, q) for q, idx in ((a2, i), (b2, j)))
    if sa == 0 or sb == 0:
        q, idx = (a, i) if sa == 0 else (b, j)
        return idx not in poly and point_in_polygon_2d(v2, _drop(q, axis))
    nrm = _cross([p1[k] - p0[k] for k in range(3)], [p2[k] - p0[k] for k in range(3)])
    t = sum(nrm[k] * (p0[k] - a[k]) for k in range(3)) / sum(nrm[k] * (b[k] - a[k]) for k in range(3))
    hit = tuple(a[k] + t * (b[k] - a[k]) for k in range(3))
    return point_in_polygon_2d(v2, _drop(hit, axis))


def _overlapping_pairs(boxes):
    """Index pairs with overlapping closed AABBs (sweep over x)."""
    order = sorted(range(len(boxes)), key=lambda k: boxes[k][0][0])
    active = []
    for k in order:
        lo, hi = boxes[k]
        active = [m for m in active if boxes[m][1][0] >= lo[0]]
        for m in active:
            mlo, mhi = boxes[m]
            if all(mlo[d] <= hi[d] and lo[d] <= mhi[d] for d in range(3)):
                yield (min(k, m), max(k, m))
        active.append(k)


FAST_MIN_FEATURES = 256    # below this the exact path is fast enough


def _exact_pair(plc: PLC, u: int, v: int) -> bool:
    """The exact pair test of the final validate loop (features numbered
    segments first, then polygons)."""
    nseg = len(plc.segments)
    if v < nseg:
        (i, j), (k, l) = plc.segments[u], plc.segments[v]
        return _segs_conflict(plc.points[i], plc.points[j], plc.points[k], plc.points[l])
    if u < nseg:
        return _seg_poly_conflict(plc.points, plc.segments[u], plc.polygons[v - nseg])
    return False


def validate(plc: PLC, fast: bool = None) -> list:
    """Every invariant violation as (code, detail); [] means valid.
    Same checks and codes as plc.py:267-383.  Large inputs are first offered
    to the vectorised certifier (setup_fast.py); anything it cannot certify
    valid goes through the exact path below."""
    if fast is None:
        fast = len(plc.segments) + len(plc.polygons) >= FAST_MIN_FEATURES
    if fast and plc.points:
        from .setup_fast import certify_valid
        if certify_valid(plc, lambda u, v: _exact_pair(plc, u, v)):
            return []
    out = []
    npts = len(plc.points)
    first = {}
    for idx, p in enumerate(plc.points):
        if not all(math.isfinite(c) for c in p):
            out.append(("nonfinite-point", idx))
        elif p in first:
            out.append(("duplicate-point", (first[p], idx)))
        else:
            first[p] = idx
    edges = set()
    for sidx, (i, j) in enumerate(plc.segments):
        if not (0 <= i < npts and 0 <= j < npts):
            out.append(("segment-bad-index", sidx))
        elif i == j or plc.points[i] == plc.points[j]:
            out.append(("segment-zero-length", sidx))
        elif (min(i, j), max(i, j)) in edges:
            out.append(("segment-duplicate", sidx))
        else:
            edges.add((min(i, j), max(i, j)))
    for pidx, poly in enumerate(plc.polygons):
        n = len(poly)
        if n < 3:
            out.append(("polygon-too-few-vertices", pidx))
            continue
        if not all(0 <= v < npts for v in poly):
            out.append(("polygon-bad-index", pidx))
            continue
        if len(set(poly)) != n:
            out.append(("polygon-repeated-vertex", pidx))
            continue
        vf = [_F(plc.points[v]) for v in poly]
        base = next(((vf[0], vf[1], vf[k]) for k in range(2, n) if not _collinear(vf[0], vf[1], vf[k])), None)
        if base is None:
            out.append(("polygon-degenerate", pidx))
            continue
        if any(_o3(*base, v) != 0 for v in vf):
            out.append(("polygon-non-planar", pidx))
            continue
        missing = [(min(poly[k], poly[(k + 1) % n]), max(poly[k], poly[(k + 1) % n]))
                   for k in range(n) if (min(poly[k], poly[(k + 1) % n]), max(poly[k], poly[(k + 1) % n])) not in edges]
        if missing:
            out.append(("polygon-edge-not-in-segments", (pidx, missing)))
            continue
        if n > 3:
            axis = _proj_axis([plc.points[v] for v in poly])
            v2 = [_drop(v, axis) for v in vf]
            simple = True
            for u in range(n):
                for w in range(u + 2, n):
                    if u == 0 and w == n - 1:
                        continue
                    if _segs_touch_2d(v2[u], v2[(u + 1) % n], v2[w], v2[(w + 1) % n], set()):
                        simple = False
            if not simple:
                out.append(("polygon-not-simple", pidx))
    if out or not plc.points:
        return out
    pts = points_array(plc)
    boxes = []
    for (i, j) in plc.segments:
        boxes.append((np.minimum(pts[i], pts[j]), np.maximum(pts[i], pts[j])))
    for poly in plc.polygons:
        q = pts[list(poly)]
        boxes.append((q.min(axis=0), q.max(axis=0)))
    nseg = len(plc.segments)
    for u, v in _overlapping_pairs(boxes):
        if v < nseg:
            (i, j), (k, l) = plc.segments[u], plc.segments[v]
            if _segs_conflict(plc.points[i], plc.points[j], plc.points[k], plc.points[l]):
                out.append(("segment-segment-intersection", (u, v)))
        elif u < nseg:
            if _seg_poly_conflict(plc.points, plc.segments[u], plc.polygons[v - nseg]):
                out.append(("segment-polygon-intersection", (u, v - nseg)))
    return out


def unit_cube() -> PLC:
    """8 corners (index = x + 2y + 4z), 12 sorted edges, 6 squares; identical
    to plc.py:386-408."""
    pts = [(float(i & 1), float((i >> 1) & 1), float((i >> 2) & 1)) for i in range(8)]

    def c(x, y, z):
        return x + 2 * y + 4 * z

    quads = [
        (c(0, 0, 0), c(1, 0, 0), c(1, 1, 0), c(0, 1, 0)),
        (c(0, 0, 1), c(0, 1, 1), c(1, 1, 1), c(1, 0, 1)),
        (c(0, 0, 0), c(0, 0, 1), c(1, 0, 1), c(1, 0, 0)),
        (c(0, 1, 0), c(1, 1, 0), c(1, 1, 1), c(0, 1, 1)),
        (c(0, 0, 0), c(0, 1, 0), c(0, 1, 1), c(0, 0, 1)),
        (c(1, 0, 0), c(1, 0, 1), c(1, 1, 1), c(1, 1, 0)),
    ]
    edges = sorted({(min(q[k], q[(k + 1) % 4]), max(q[k], q[(k + 1) % 4])) for q in quads for k in range(4)})
    return PLC(points=pts, segments=edges, polygons=quads)


# ---------------------------------------------------------------------------
# domain closure (refine.py:421-506)

def hull_simplices(plc: PLC):
    """Triangles of the convex hull of the points (scipy Qhull, as the
    reference's _hull_covered uses, refine.py:455-459), or None.

    With polygons, the hull of their vertices is built first; points strictly
    inside its inscribed ball (with a relative margin) cannot be hull
    vertices and are left out of the final hull computation (C4: 1M interior
    points, 122k surface vertices)."""
    from scipy.spatial import ConvexHull, QhullError

    P = points_array(plc)
    try:
        if plc.polygons and len(P) > 10000:
            sv = np.unique(polygon_index_array(plc))
            if len(sv) >= 4:
                h0 = ConvexHull(P[sv])
                ctr = P[sv][h0.vertices].mean(axis=0)
                r_in = float(np.min(-(h0.equations[:, :3] @ ctr + h0.equations[:, 3])))
                scale = float(np.max(np.abs(P[sv] - ctr)))
                if r_in > 1e-6 * scale:
                    d = np.sqrt(np.sum((P - ctr) ** 2, axis=1))
                    keep = d >= r_in * (1.0 - 1e-9) - 1e-12 * scale
                    keep[sv] = True
                    idx = np.flatnonzero(keep)
                    if len(idx) == len(sv):
                        return sv[h0.simplices]
                    if len(idx) < len(P):
                        return idx[ConvexHull(P[idx]).simplices]
        return ConvexHull(P).simplices
    except QhullError:
        return None


def hull_axis_aligned(plc: PLC, simplices) -> bool:
    """True when every hull triangle lies in a coordinate plane (its three
    vertices share one coordinate exactly)."""
    tri = points_array(plc)[np.asarray(simplices)]
    same = (tri[:, 0, :] == tri[:, 1, :]) & (tri[:, 0, :] == tri[:, 2, :])
    return bool(np.all(np.any(same, axis=1)))


def hull_covered(plc: PLC, simplices=None) -> bool:
    """True when the polygons tile the convex hull of the points.  Same
    decision as refine.py:421-459, indexed by vertex instead of scanning all
    polygons per hull triangle."""
    if simplices is None:
        simplices = hull_simplices(plc)
    if simplices is None:
        return False
    from .setup_fast import certify_hull_covered
    if certify_hull_covered(plc, simplices):
        return True
    by_vertex = {}
    for pid, poly in enumerate(plc.polygons):
        for v in poly:
            by_vertex.setdefault(v, []).append(pid)
    cache = {}
    for simplex in simplices:
        tri = [int(v) for v in simplex]
        cands = set(by_vertex.get(tri[0], ()))
        for v in tri[1:]:
            cands &= set(by_vertex.get(v, ()))
        ok = False
        for pid in sorted(cands):
            poly = plc.polygons[pid]
            if pid not in cache:
                axis = _proj_axis([plc.points[v] for v in poly])
                keep = [k for k in range(3) if k != axis]
                cache[pid] = (keep, [(plc.points[v][keep[0]], plc.points[v][keep[1]]) for v in poly])
            keep, p2 = cache[pid]
            cx = sum(Fraction(plc.points[v][keep[0]]) for v in tri) / 3
            cy = sum(Fraction(plc.points[v][keep[1]]) for v in tri) / 3
            if point_in_polygon_2d(p2, (cx, cy)):
                ok = True
                break
        if not ok:
            return False
    return True


def augment_with_box(plc: PLC) -> PLC:
    """Wrap the points in an axis-aligned box padded by 0.25*diag unless the
    polygons already tile the hull (refine.py:462-506); corners, edges and
    faces are appended after the input features in the same order.

    One deliberate difference: a hull tiled by polygons that are not all in
    coordinate planes (a sphere's triangles) gets the box too.  The reference
    boxes the domain precisely so that boundary Steiner points round exactly
    onto their facet planes (refine.py:466-473); on an oblique hull facet a
    rounded midpoint lands a few ulps outside the hull, and its ghost cavity
    need not star.  The reference never reaches that case (it stops on
    oblique facets in Tri2D), so every input it refines is
    unaffected.  Such a box is marked (``box_for_oblique_hull``): bulk
    construction then inserts its corners first (prepare.py), since a corner
    inserted after the curved hull would see a quarter of it at once."""
    for_oblique = False
    if plc.polygons:
        hs = hull_simplices(plc)
        oblique_box = os.environ.get("GQM3D_OBLIQUE_BOX", "1") != "0"   # experiments: 0 = reference rule
        if hs is not None and hull_covered(plc, hs):
            if not oblique_box or hull_axis_aligned(plc, hs):
                return plc
            for_oblique = True
    lo, hi = bounding_box(plc)
    pad = 0.25 * math.dist(lo, hi)
    lo = tuple(x - pad for x in lo)
    hi = tuple(x + pad for x in hi)
    n = len(plc.points)
    corners = [(hi[0] if i else lo[0], hi[1] if j else lo[1], hi[2] if k else lo[2])
               for i in (0, 1) for j in (0, 1) for k in (0, 1)]
    faces = []
    for axis in range(3):
        for side in (0, 1):
            quad = []
            for a, b in ((0, 0), (0, 1), (1, 1), (1, 0)):
                bits = [0, 0, 0]
                bits[axis], bits[(axis + 1) % 3], bits[(axis + 2) % 3] = side, a, b
                quad.append(n + 4 * bits[0] + 2 * bits[1] + bits[2])
            faces.append(tuple(quad))
    edges = sorted({(min(q[k], q[(k + 1) % 4]), max(q[k], q[(k + 1) % 4])) for q in faces for k in range(4)})
    out = PLC._normalised(list(plc.points) + [tuple(float(x) for x in q) for q in corners],
                          list(plc.segments) + [tuple(int(i) for i in e) for e in edges],
                          list(plc.polygons) + [tuple(int(i) for i in f) for f in faces])
    out.__dict__["box_for_oblique_hull"] = for_oblique
    return out
