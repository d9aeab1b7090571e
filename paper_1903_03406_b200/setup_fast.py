"""Vectorised certification of large PLCs (native setup).

``validate`` (plc.py:267-383 of the reference), the hull-coverage test of the
domain closure (refine.py:421-459) and the facet projection axes
(facets.py:256-273) decide everything in exact rational arithmetic, one
feature pair at a time -- hours of Python for the 200k-triangle C4 input.

This module reaches the same decisions for the common case in numpy:

* a floating-point filter with a rigorous error bound decides each predicate
  when it can (orientation signs, collinearity, normal components); entries
  it cannot certify are handed to the exact Fraction code of ``plc.py``;
* candidate feature pairs come from a uniform grid over the bounding boxes
  instead of a Python sweep; a pair is then cleared by the filter or checked
  by the exact pair test;
* whenever anything looks invalid, the caller falls back to the exact
  reference-order implementation, so the reported violations (and their
  order) are always the exact path's.

Functions return ``True`` ("certified") or ``None`` ("not certified, use the
exact path"); they never report a violation themselves.
"""

from __future__ import annotations

import os

import numpy as np

_EPS = 2.0 ** -53
# |fl(expr) - expr| <= bound * (sum of |products|) for a 2x2 / 3x3 determinant
# evaluated from rounded differences (conservative: 16 eps for the cross
# products of differences, 32 eps for the triple product).
_CROSS_B = 16.0 * _EPS
_O3_B = 32.0 * _EPS


def _cross_with_bound(u, v):
    """Cross products of rows and a per-component absolute error bound."""
    t = np.stack([u[:, 1] * v[:, 2], u[:, 2] * v[:, 1],
                  u[:, 2] * v[:, 0], u[:, 0] * v[:, 2],
                  u[:, 0] * v[:, 1], u[:, 1] * v[:, 0]], axis=1)
    c = np.stack([t[:, 0] - t[:, 1], t[:, 2] - t[:, 3], t[:, 4] - t[:, 5]], axis=1)
    err = _CROSS_B * np.stack([np.abs(t[:, 0]) + np.abs(t[:, 1]), np.abs(t[:, 2]) + np.abs(t[:, 3]),
                               np.abs(t[:, 4]) + np.abs(t[:, 5])], axis=1)
    return c, err


def orient3d_filtered(a, b, c, d):
    """sign(det[b-a, c-a, d-a]) as in plc._o3; 2 where the filter is unsure."""
    u, v, w = b - a, c - a, d - a
    m0 = v[:, 1] * w[:, 2]; m1 = v[:, 2] * w[:, 1]
    m2 = v[:, 0] * w[:, 2]; m3 = v[:, 2] * w[:, 0]
    m4 = v[:, 0] * w[:, 1]; m5 = v[:, 1] * w[:, 0]
    det = u[:, 0] * (m0 - m1) - u[:, 1] * (m2 - m3) + u[:, 2] * (m4 - m5)
    perm = (np.abs(u[:, 0]) * (np.abs(m0) + np.abs(m1)) + np.abs(u[:, 1]) * (np.abs(m2) + np.abs(m3))
            + np.abs(u[:, 2]) * (np.abs(m4) + np.abs(m5)))
    s = np.sign(det).astype(np.int8)
    s[~(np.abs(det) > _O3_B * perm)] = 2
    return s


def orient3d_resolved(a, b, c, d):
    """orient3d_filtered with the unsure entries decided exactly (integer
    arithmetic on the scaled mantissas, exactnp._o3d_exact): same sign as
    plc._o3 everywhere."""
    from .exactnp import _o3d_exact

    s = orient3d_filtered(a, b, c, d)
    for k in np.flatnonzero(s == 2):
        s[k] = _o3d_exact(a[k], b[k], c[k], d[k])
    return s


# ---------------------------------------------------------------------------
# candidate pairs with overlapping closed AABBs (plc._overlapping_pairs)

def overlapping_pairs(lo: np.ndarray, hi: np.ndarray, max_span: int = 3):
    """All index pairs (u < v) whose closed boxes overlap, via grid binning."""
    n = len(lo)
    if n < 2:
        return np.zeros((0, 2), dtype=np.int64)
    ext = hi - lo
    glo = lo.min(axis=0)
    span = np.maximum(hi.max(axis=0) - glo, 1e-300)
    cell = max(float(np.median(ext.max(axis=1))) * 2.0, float(span.max()) / 256.0, 1e-300)
    G = np.minimum(np.ceil(span / cell).astype(np.int64) + 1, 1 << 20)
    i0 = np.clip(np.floor((lo - glo) / cell).astype(np.int64), 0, G - 1)
    i1 = np.clip(np.floor((hi - glo) / cell).astype(np.int64), 0, G - 1)
    spans = i1 - i0
    big = np.flatnonzero((spans >= max_span).any(axis=1))
    small = np.flatnonzero(~(spans >= max_span).any(axis=1))
    keys, ids = [], []
    for dx in range(max_span):
        for dy in range(max_span):
            for dz in range(max_span):
                m = small[(spans[small, 0] >= dx) & (spans[small, 1] >= dy) & (spans[small, 2] >= dz)]
                if len(m) == 0:
                    continue
                cx, cy, cz = i0[m, 0] + dx, i0[m, 1] + dy, i0[m, 2] + dz
                keys.append((cx * G[1] + cy) * G[2] + cz)
                ids.append(m)
    pairs = []
    if keys:
        key = np.concatenate(keys)
        idv = np.concatenate(ids)
        o = np.argsort(key, kind="stable")
        key, idv = key[o], idv[o]
        # pairs inside each cell: shift the sorted list against itself
        s = 1
        while s < len(key):
            same = key[s:] == key[:-s]
            if not same.any():
                break
            a, b = idv[:-s][same], idv[s:][same]
            pairs.append(np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1))
            s += 1
    for k in big:   # boxes spanning many cells: tested against everything
        ov = np.flatnonzero(np.all((lo <= hi[k]) & (lo[k] <= hi), axis=1))
        ov = ov[ov != k]
        pairs.append(np.stack([np.minimum(ov, k), np.maximum(ov, k)], axis=1))
    if not pairs:
        return np.zeros((0, 2), dtype=np.int64)
    P = np.concatenate(pairs).astype(np.int64)
    key = np.sort(P[:, 0] * n + P[:, 1])
    key = key[np.concatenate([[True], key[1:] != key[:-1]])]
    P = np.stack([key // n, key % n], axis=1)
    u, v = P[:, 0], P[:, 1]
    ok = np.all((lo[u] <= hi[v]) & (lo[v] <= hi[u]), axis=1)
    return P[ok]


# ---------------------------------------------------------------------------
# validate (plc.py:267-383)

def has_duplicate_points(P) -> bool:
    """Equal coordinate triples (as the reference's tuple comparison sees
    them: -0.0 == 0.0).  A 64-bit hash sort finds the candidates, an exact
    comparison confirms them."""
    if len(P) < 2:
        return False
    k = np.ascontiguousarray(P + 0.0).view(np.uint64).reshape(-1, 3)
    h = (k[:, 0] * np.uint64(0x9E3779B97F4A7C15)) ^ (k[:, 1] * np.uint64(0xC2B2AE3D27D4EB4F)) \
        ^ (k[:, 2] * np.uint64(0x165667B19E3779F9))
    o = np.argsort(h, kind="stable")
    hs = h[o]
    same = np.flatnonzero(hs[1:] == hs[:-1])
    if len(same) == 0:
        return False
    cand = np.unique(np.concatenate([o[same], o[same + 1]]))
    Q = P[cand]
    q = Q[np.lexsort((Q[:, 2], Q[:, 1], Q[:, 0]))]
    return bool(np.any(np.all(q[1:] == q[:-1], axis=1)))


def _native_pairs(P, S, tri):
    """(status, undecided pairs) from the device certifier, or None without a
    usable GPU / library (then the numpy path decides)."""
    if os.environ.get("GQM3D_HOST_SETUP") == "1":
        return None
    try:
        from . import _native
        from .refine import default_device
        return _native.certify_pairs(P, S, tri, device=default_device())
    except Exception:
        return None


def certify_valid(plc, exact_pair) -> bool | None:
    """True when the PLC has no violation; None when the exact path must
    decide.  ``exact_pair(u, v)`` runs the exact pair test of plc.validate
    (seg-seg or seg-polygon, indices in the combined feature numbering)."""
    from .plc import _F, _collinear

    from .plc import points_array
    P = points_array(plc)
    npts = len(P)
    if npts == 0 or not np.all(np.isfinite(P)):
        return None
    if has_duplicate_points(P):
        return None
    S = np.asarray(plc.segments, dtype=np.int64).reshape(-1, 2)
    if len(S):
        if S.min() < 0 or S.max() >= npts or np.any(S[:, 0] == S[:, 1]):
            return None
        if np.any(np.all(P[S[:, 0]] == P[S[:, 1]], axis=1)):
            return None
        ek = np.minimum(S[:, 0], S[:, 1]) * npts + np.maximum(S[:, 0], S[:, 1])
        ek_sorted = np.sort(ek)
        if np.any(ek_sorted[1:] == ek_sorted[:-1]):
            return None
    else:
        ek_sorted = np.zeros(0, dtype=np.int64)
    polys = plc.polygons
    tri = np.array([p for p in polys if len(p) == 3], dtype=np.int64).reshape(-1, 3)
    if len(tri) != len(polys):
        return None                      # general polygons: exact path
    if len(tri):
        if tri.min() < 0 or tri.max() >= npts:
            return None
        if np.any((tri[:, 0] == tri[:, 1]) | (tri[:, 1] == tri[:, 2]) | (tri[:, 0] == tri[:, 2])):
            return None
        # non-degenerate: a certainly nonzero normal component, else exact
        nrm, err = _cross_with_bound(P[tri[:, 1]] - P[tri[:, 0]], P[tri[:, 2]] - P[tri[:, 0]])
        unsure = np.flatnonzero(~np.any(np.abs(nrm) > err, axis=1))
        for k in unsure:
            a, b, c = (_F(plc.points[int(v)]) for v in tri[k])
            if _collinear(a, b, c):
                return None
        # every edge is a segment
        for x, y in ((0, 1), (1, 2), (2, 0)):
            key = np.minimum(tri[:, x], tri[:, y]) * npts + np.maximum(tri[:, x], tri[:, y])
            pos = np.searchsorted(ek_sorted, key)
            pos = np.minimum(pos, max(len(ek_sorted) - 1, 0))
            if len(ek_sorted) == 0 or np.any(ek_sorted[pos] != key):
                return None
    # feature pairs with overlapping boxes: on the device when there is one
    # (exact predicates, gq_certify_pairs), else the vectorised filter below
    native = _native_pairs(P, S, tri)
    if native is not None:
        status, undecided = native
        if status != 0:
            return None
        for x, y in undecided.tolist():
            if exact_pair(int(x), int(y)):
                return None
        return True
    nseg = len(S)
    lo = np.concatenate([np.minimum(P[S[:, 0]], P[S[:, 1]]), P[tri].min(axis=1)]) if len(tri) else \
        np.minimum(P[S[:, 0]], P[S[:, 1]])
    hi = np.concatenate([np.maximum(P[S[:, 0]], P[S[:, 1]]), P[tri].max(axis=1)]) if len(tri) else \
        np.maximum(P[S[:, 0]], P[S[:, 1]])
    pairs = overlapping_pairs(lo, hi)
    if len(pairs) == 0:
        return True
    u, v = pairs[:, 0], pairs[:, 1]
    ss = v < nseg                                     # both segments (u < v)
    sp = (u < nseg) & (v >= nseg)                     # segment u, polygon v - nseg
    unsure = []
    # -- segment / segment
    U, V = u[ss], v[ss]
    if len(U):
        a, b, c, d = S[U, 0], S[U, 1], S[V, 0], S[V, 1]
        share = (a == c) | (a == d) | (b == c) | (b == d)
        # disjoint endpoints: not coplanar => no conflict (plc._segs_conflict)
        o = np.zeros(len(U), dtype=np.int8)
        ns = np.flatnonzero(~share)
        o[ns] = orient3d_resolved(P[a[ns]], P[b[ns]], P[c[ns]], P[d[ns]])
        clear = ~share & (o != 0)
        # one shared endpoint: conflict only if the three points are collinear
        sh = np.flatnonzero(share)
        if len(sh):
            pa, pb = P[a[sh]], P[b[sh]]
            other = np.where((c[sh] == a[sh]) | (c[sh] == b[sh]), d[sh], c[sh])
            nrm, err = _cross_with_bound(pb - pa, P[other] - pa)
            clear[sh] = np.any(np.abs(nrm) > err, axis=1)
        unsure += list(zip(U[~clear].tolist(), V[~clear].tolist()))
    # -- segment / triangle
    U, V = u[sp], v[sp]
    if len(U):
        i, j = S[U, 0], S[U, 1]
        T = tri[V - nseg]
        in_i = (T == i[:, None]).any(axis=1)
        in_j = (T == j[:, None]).any(axis=1)
        edge = in_i & in_j                           # a side of the triangle
        p0, p1, p2 = P[T[:, 0]], P[T[:, 1]], P[T[:, 2]]
        # the shared vertex of a triangle is an exact zero; the rest exactly
        sa = np.zeros(len(U), dtype=np.int8)
        sb = np.zeros(len(U), dtype=np.int8)
        ki, kj = np.flatnonzero(~in_i & ~edge), np.flatnonzero(~in_j & ~edge)
        sa[ki] = orient3d_resolved(p0[ki], p1[ki], p2[ki], P[i[ki]])
        sb[kj] = orient3d_resolved(p0[kj], p1[kj], p2[kj], P[j[kj]])
        certain = np.ones(len(U), dtype=bool)
        same_side = certain & (sa * sb > 0)
        # one endpoint on the plane: that endpoint is a vertex of the triangle
        # and the other one is off the plane -> no conflict (plc._seg_poly_conflict)
        touch = certain & (((sa == 0) & in_i & (sb != 0)) | ((sb == 0) & in_j & (sa != 0)))
        # a proper plane crossing hits the closed triangle iff the orientations
        # of the line against its three sides are not of strictly mixed sign
        cross = np.flatnonzero(certain & (sa * sb < 0) & ~edge & ~in_i & ~in_j)
        miss = np.zeros(len(U), dtype=bool)
        if len(cross):
            pa, pb = P[i[cross]], P[j[cross]]
            q = [p0[cross], p1[cross], p2[cross]]
            o = np.stack([orient3d_resolved(pa, pb, q[k], q[(k + 1) % 3]) for k in range(3)], axis=1)
            miss[cross] = ((o == 1).any(axis=1)) & ((o == -1).any(axis=1))
        clear = edge | same_side | touch | miss
        unsure += list(zip(U[~clear].tolist(), V[~clear].tolist()))
    for x, y in unsure:
        if exact_pair(int(x), int(y)):
            return None
    return True


# ---------------------------------------------------------------------------
# hull coverage (refine.py:421-459) and facet axes (facets.py:256-273)

def certify_hull_covered(plc, hull_simplices) -> bool | None:
    """True when every hull triangle is one of the (triangular) polygons --
    its centroid then lies strictly inside that polygon; None otherwise."""
    polys = plc.polygons
    if not polys or any(len(p) != 3 for p in polys):
        return None
    n = len(plc.points)
    T = np.sort(np.asarray(polys, dtype=np.int64), axis=1)
    H = np.sort(np.asarray(hull_simplices, dtype=np.int64), axis=1)
    kt = (T[:, 0] * n + T[:, 1]) * n + T[:, 2]
    kh = (H[:, 0] * n + H[:, 1]) * n + H[:, 2]
    return True if np.all(np.isin(kh, kt)) else None


def facet_axes(plc):
    """(f, 2) projection axes for triangles with certified normals; rows that
    need the exact path are returned as -1."""
    polys = plc.polygons
    out = np.full((len(polys), 2), -1, dtype=np.int32)
    from .plc import points_array, polygon_index_array
    flat = polygon_index_array(plc)
    if len(flat) == 3 * len(polys) and all(len(p) == 3 for p in polys[:1]):   # uniform: all triangles
        idx = np.arange(len(polys), dtype=np.int64)
        T = flat.reshape(-1, 3)
    else:
        idx = np.array([k for k, p in enumerate(polys) if len(p) == 3], dtype=np.int64)
        T = np.asarray([polys[k] for k in idx], dtype=np.int64).reshape(-1, 3)
    if len(idx) == 0:
        return out
    P = points_array(plc)
    nrm, err = _cross_with_bound(P[T[:, 1]] - P[T[:, 0]], P[T[:, 2]] - P[T[:, 0]])
    mag = np.abs(nrm)
    best = np.argmax(mag, axis=1)                    # first on ties, like plc._proj_axis
    r = np.arange(len(T))
    ok = mag[r, best] > err[r, best]
    for k in range(3):                               # strictly larger than the others, certainly
        other = k != best
        ok &= ~other | (mag[r, best] - err[r, best] > mag[:, k] + err[:, k])
    # projected signed area has the sign of +n0, -n1, +n2 for axis 0, 1, 2
    sgn = np.sign(nrm[r, best]) * np.where(best == 1, -1.0, 1.0)
    ij = np.array([[1, 2], [0, 2], [0, 1]], dtype=np.int32)[best]
    ij = np.where((sgn < 0)[:, None], ij[:, ::-1], ij)
    out[idx[ok]] = ij[ok]
    return out
