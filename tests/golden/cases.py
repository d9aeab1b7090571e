"""Golden-case builders (no reference import: safe on the GPU box)."""

import hashlib
import json

from paper_1903_03406_b200 import synth

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
}


def tet_hash(tv_rows) -> str:
    rows = sorted(tuple(sorted(int(v) for v in r)) for r in tv_rows)
    return hashlib.sha1(json.dumps(rows).encode()).hexdigest()
