"""Host-side setup shared by the GPU path and the test oracle.

``refine()`` in the reference validates the PLC, closes the domain with a
padded box and shuffles the insertion order before any meshing happens
(/root/reference/pkg/src/tetrefine/refine.py:523-531, mesh.py:873-880).
``prepare`` does exactly that and flattens the result into the plain arrays
the C ABI takes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import AllCoplanar, DuplicatePoint, InvalidPLC
from .plc import PLC, augment_with_box, points_array, validate


@dataclass
class Prepared:
    plc: PLC              # augmented PLC
    n_input: int          # points of the caller's PLC (origin 0)
    points: np.ndarray    # (n,3) float64, C-contiguous
    segments: np.ndarray  # (m,2) int32
    poly_off: np.ndarray  # (f+1,) int32
    poly_idx: np.ndarray  # (sum,) int32
    order: np.ndarray     # (n,) int32 insertion order
    setup_s: float = 0.0


def shuffle_order(n: int, seed: int) -> np.ndarray:
    """mesh.py:878-880: list(range(n)) shuffled in place by default_rng(seed).
    Generator.shuffle draws the same Fisher-Yates sequence for a 1-D array as
    for a list (tests/test_host.py checks the two agree), ~4x faster."""
    order = np.arange(n, dtype=np.int64)
    np.random.default_rng(seed).shuffle(order)
    return order.astype(np.int32)


def insertion_order(aug: PLC, n_input: int, n: int, seed: int) -> np.ndarray:
    """The reference's shuffled order (mesh.py:878-880); for a box added
    around an oblique hull (plc.augment_with_box) its 8 corners go first and
    the input points follow in the shuffled order of the input alone."""
    if not aug.__dict__.get("box_for_oblique_hull"):
        return shuffle_order(n, seed)
    return np.concatenate([np.arange(n_input, n, dtype=np.int32), shuffle_order(n_input, seed)])


def prepare(plc: PLC, seed: int = 0, check: bool = True) -> Prepared:
    import time

    t0 = time.perf_counter()
    if check:
        violations = validate(plc)
        if violations:
            raise InvalidPLC(violations)
    aug = augment_with_box(plc)
    if aug is plc:
        pts = np.ascontiguousarray(points_array(plc))
    else:   # input points (converted once already) + the 8 box corners
        pts = np.ascontiguousarray(np.concatenate([points_array(plc),
                                                   np.asarray(aug.points[len(plc.points):], dtype=np.float64).reshape(-1, 3)]))
    if len(pts) < 4:
        raise AllCoplanar("need at least 4 points")
    # validate() already rejects duplicate input points, and box corners lie
    # 0.25*diag outside the input bbox, so the sort is only needed unchecked
    if not check:
        q = pts[np.lexsort((pts[:, 2], pts[:, 1], pts[:, 0]))]
        if len(q) > 1 and np.any(np.all(q[1:] == q[:-1], axis=1)):
            raise DuplicatePoint("duplicate input points")
    segs = np.ascontiguousarray(np.asarray(aug.segments, dtype=np.int32).reshape(-1, 2))
    off = [0]
    idx = []
    for poly in aug.polygons:
        idx.extend(poly)
        off.append(len(idx))
    return Prepared(plc=aug, n_input=len(plc.points), points=pts, segments=segs,
                    poly_off=np.asarray(off, dtype=np.int32), poly_idx=np.asarray(idx, dtype=np.int32),
                    order=insertion_order(aug, len(plc.points), len(pts), seed), setup_s=time.perf_counter() - t0)


def facet_keep(plc: PLC) -> np.ndarray:
    """Projection axes (i, j) of every polygon, ordered so the projected
    boundary is counterclockwise (facets.py:256-273, exact)."""
    from fractions import Fraction

    from .plc import _proj_axis

    from .setup_fast import facet_axes

    out = facet_axes(plc)          # triangles with a certified normal (vectorised)
    cache = {}
    for pid in np.flatnonzero(out[:, 0] < 0).tolist():
        poly = plc.polygons[pid]
        pts = [plc.points[v] for v in poly]
        axis = _proj_axis(pts)
        i, j = [k for k in range(3) if k != axis]
        # exact signed area of the projected cycle
        tot = Fraction(0)
        n = len(pts)
        for k in range(n):
            x0, y0 = Fraction(pts[k][i]), Fraction(pts[k][j])
            x1, y1 = Fraction(pts[(k + 1) % n][i]), Fraction(pts[(k + 1) % n][j])
            tot += x0 * y1 - x1 * y0
        if tot < 0:
            i, j = j, i
        out[pid] = (i, j)
        # (non-convex polygons: the device keeps a 2D triangle as a subface only
        # when its centroid is inside the polygon, facets.py:278-291)
    del cache
    return out
