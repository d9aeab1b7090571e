"""Golden-case builders (no reference import: safe on the GPU box)."""

import hashlib
import json

from paper_1903_03406_b200 import synth

def _lshape(n: int, seed: int):
    """Unit cube + n points + one non-convex (L-shaped) hexagon in z = 0.5:
    the reference keeps only 2D triangles whose centroid is inside it."""
    from paper_1903_03406_b200 import PLC
    base = synth.cube_points(n, seed)
    k = len(base.points)
    L = [(0.2, 0.2, 0.5), (0.8, 0.2, 0.5), (0.8, 0.5, 0.5), (0.5, 0.5, 0.5), (0.5, 0.8, 0.5), (0.2, 0.8, 0.5)]
    segs = [(k + i, k + (i + 1) % 6) for i in range(6)]
    return PLC(points=list(base.points) + L, segments=list(base.segments) + segs,
               polygons=list(base.polygons) + [tuple(range(k, k + 6))])


CASES = {
    # name: (builder, B)
    "cube0": (lambda: synth.cube_points(0, 0), 2.0),
    "cube100": (lambda: synth.cube_points(100, 0), 2.0),
    "cube300": (lambda: synth.cube_points(300, 0), 2.0),
    "c1": (lambda: synth.cube_points(1000, 0), 2.0),
    "seg1000": (lambda: synth.segments_cloud(1000, 10, 0), 1.6),
    "rect600": (lambda: synth.generate(synth.SynthSpec(600, 0.01, "cube", 0)), 1.6),
    "tri500": (lambda: synth.triangles_cloud(500, 5, 0), 1.4),
    "oblique500": (lambda: synth.triangles_cloud(500, 5, 0, snapped=False), 1.6),
    "lshape400": (lambda: _lshape(400, 5), 1.8),
}


def tet_hash(tv_rows) -> str:
    rows = sorted(tuple(sorted(int(v) for v in r)) for r in tv_rows)
    return hashlib.sha1(json.dumps(rows).encode()).hexdigest()
