"""Seeded synthetic PLCs for the benchmark configurations.

C1  unit cube + n uniform interior points                          (B=2.0)
C2  n uniform points + m random oblique segments (endpoints added)   (B=1.6)
C3  n points + m pairwise-disjoint triangles (axis-plane, snapped to
    a 2^-16 grid in the parity variant)                              (B=1.4)
C4  nested icospheres + torus surface + n interior ball points       (B=1.5)
C5  a batch of C1-shaped PLCs with seeds 0..K-1                      (B=1.5)

Plus ``generate(SynthSpec)``: the reference's own rectangle generator
(/root/reference/pkg/src/tetrefine/synth.py:60-107), same sampling order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import PlacementFailure
from .plc import PLC, unit_cube


def cube_points(n: int, seed: int = 0) -> PLC:
    """C1 / C5: unit cube plus n uniform points appended after the corners."""
    base = unit_cube()
    pts = np.random.default_rng(seed).uniform(0.0, 1.0, (n, 3))
    return PLC(points=list(base.points) + [tuple(p) for p in pts], segments=base.segments,
               polygons=base.polygons)


def segments_cloud(n: int, m: int, seed: int = 0) -> PLC:
    """C2: n uniform points in the unit cube + m random segments: start
    a ~ U[0.1,0.9]^3, direction uniform on the sphere, length U[0.01,0.1]."""
    rng = np.random.default_rng(seed)
    pts = [tuple(p) for p in rng.uniform(0.0, 1.0, (n, 3))]
    segs = []
    for _ in range(m):
        a = rng.uniform(0.1, 0.9, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        b = a + d * rng.uniform(0.01, 0.1)
        i = len(pts)
        pts.append(tuple(a))
        pts.append(tuple(b))
        segs.append((i, i + 1))
    return PLC(points=pts, segments=segs, polygons=[])


def triangles_cloud(n: int, m: int, seed: int = 0, snapped: bool = True) -> PLC:
    """C3: n uniform points + m triangles with pairwise-disjoint AABBs.
    snapped=True: axis-plane triangles on a 2^-16 grid (the reference-robust
    parity variant); False: oblique triangles (stress variant)."""
    rng = np.random.default_rng(seed)
    g = 2.0 ** -16
    tris = []
    boxes = []
    tries = 0
    while len(tris) < m:
        tries += 1
        if tries > 1000 * max(1, m):
            raise PlacementFailure("triangle placement exhausted")
        c = rng.uniform(0.1, 0.9, 3)
        size = rng.uniform(0.01, 0.05)
        ang = rng.uniform(0.0, 2 * np.pi) + np.array([0.0, 2 * np.pi / 3, 4 * np.pi / 3]) \
            + rng.uniform(-0.2, 0.2, 3)
        rad = size * rng.uniform(0.9, 1.1, 3)
        if snapped:
            axis = int(rng.integers(3))
            u, w = [k for k in range(3) if k != axis]
            q = np.zeros((3, 3))
            q[:, u] = rad * np.cos(ang)
            q[:, w] = rad * np.sin(ang)
            v = np.round((c + q) / g) * g
        else:
            e1 = rng.normal(size=3)
            e1 /= np.linalg.norm(e1)
            e2 = np.cross(e1, rng.normal(size=3))
            e2 /= np.linalg.norm(e2)
            v = c + (rad * np.cos(ang))[:, None] * e1 + (rad * np.sin(ang))[:, None] * e2
        # well-shaped only: every angle >= 50 degrees (no segment cascades)
        angs = []
        for k in range(3):
            a, b = v[(k + 1) % 3] - v[k], v[(k + 2) % 3] - v[k]
            angs.append(np.degrees(np.arccos(np.dot(a, b) / np.linalg.norm(a) / np.linalg.norm(b))))
        if min(angs) < 50.0:
            continue
        lo, hi = v.min(axis=0) - 1e-3, v.max(axis=0) + 1e-3
        if any(np.all(lo <= bh) and np.all(bl <= hi) for bl, bh in boxes):
            continue
        boxes.append((lo, hi))
        tris.append(v)
    pts = rng.uniform(0.0, 1.0, (n, 3))
    # drop cloud points inside any triangle's padded box (keeps the PLC valid)
    keep = np.ones(n, dtype=bool)
    for lo, hi in boxes:
        keep &= ~np.all((pts >= lo) & (pts <= hi), axis=1)
    points = [tuple(p) for p in pts[keep]]
    segs, polys = [], []
    for v in tris:
        i = len(points)
        points.extend(tuple(x) for x in v)
        segs.extend([(i, i + 1), (i + 1, i + 2), (i, i + 2)])
        polys.append((i, i + 1, i + 2))
    return PLC(points=points, segments=segs, polygons=polys)


def _icosphere(level: int, radius: float):
    t = (1.0 + 5 ** 0.5) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.array(p, dtype=np.float64) / np.linalg.norm(p) for p in v]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
             (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        cache = {}

        def mid(a, b):
            k = (min(a, b), max(a, b))
            if k not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[k] = len(verts) - 1
            return cache[k]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    return np.array(verts) * radius, faces


def nested_surfaces(n: int, level: int = 6, torus=(200, 100), seed: int = 0) -> PLC:
    """C4: outer icosphere r=1 + inner icosphere r=0.45 + torus R=0.72,
    r=0.12 (triangulated quads) + n points uniform in the unit ball, rejecting
    points within 1e-3 of a surface."""
    rng = np.random.default_rng(seed)
    points, segs, polys = [], set(), []

    def add_mesh(V, F):
        base = len(points)
        points.extend(tuple(p) for p in V)
        for a, b, c in F:
            a, b, c = a + base, b + base, c + base
            polys.append((a, b, c))
            for u, w in ((a, b), (b, c), (c, a)):
                segs.add((min(u, w), max(u, w)))

    V, F = _icosphere(level, 1.0)
    add_mesh(V, F)
    V, F = _icosphere(level, 0.45)
    add_mesh(V, F)
    nu, nv = torus
    R, r = 0.72, 0.12
    TV = []
    for i in range(nu):
        for j in range(nv):
            u, w = 2 * np.pi * i / nu, 2 * np.pi * j / nv
            TV.append(((R + r * np.cos(w)) * np.cos(u), (R + r * np.cos(w)) * np.sin(u), r * np.sin(w)))
    TF = []
    for i in range(nu):
        for j in range(nv):
            a, b = i * nv + j, ((i + 1) % nu) * nv + j
            c, d = ((i + 1) % nu) * nv + (j + 1) % nv, i * nv + (j + 1) % nv
            TF += [(a, b, c), (a, c, d)]
    add_mesh(np.array(TV), TF)
    cloud = []
    while len(cloud) < n:
        q = rng.uniform(-1.0, 1.0, (2 * n, 3))
        rr = np.linalg.norm(q, axis=1)
        ok = (rr < 1.0 - 1e-3) & (np.abs(rr - 0.45) > 1e-3)
        rho = np.hypot(np.hypot(q[:, 0], q[:, 1]) - R, q[:, 2])
        ok &= np.abs(rho - r) > 1e-3
        cloud.extend(tuple(p) for p in q[ok][: n - len(cloud)])
    return PLC(points=points + cloud, segments=sorted(segs), polygons=polys)


CONFIGS = {
    "C1": dict(B=2.0, desc="unit-cube PLC + 1k uniform interior points"),
    "C2": dict(B=1.6, desc="100k uniform points + 1k random segments"),
    "C3": dict(B=1.4, desc="250k points + 2k disjoint triangular facets"),
    "C4": dict(B=1.5, desc="nested sphere/torus surface (~200k tris) + 1M points"),
    "C5": dict(B=1.5, desc="64 independent 50k-point cube PLCs"),
}


def config_plc(name: str, scale: float = 1.0, seed: int = 0) -> PLC:
    """PLC of a BASELINE config; ``scale`` shrinks point counts for tests."""
    if name == "C1":
        return cube_points(max(1, int(1000 * scale)), seed)
    if name == "C2":
        return segments_cloud(max(4, int(100000 * scale)), max(1, int(1000 * scale)), seed)
    if name == "C3":
        return triangles_cloud(max(4, int(250000 * scale)), max(1, int(2000 * scale)), seed)
    if name == "C4":
        return nested_surfaces(max(4, int(1000000 * scale)), seed=seed)
    if name == "C5":
        return cube_points(max(1, int(50000 * scale)), seed)
    raise ValueError(name)


# ---------------------------------------------------------------------------
# the reference's rectangle generator (synth.py:24-107)

@dataclass(frozen=True)
class SynthSpec:
    n_points: int
    gamma: float = 0.0
    distribution: str = "ball"
    seed: int = 0

    def __post_init__(self):
        if self.n_points < 4:
            raise ValueError("n_points must be at least 4")
        if self.gamma < 0:
            raise ValueError("gamma must be nonnegative")
        if self.distribution not in ("ball", "cube"):
            raise ValueError(f"unknown distribution {self.distribution!r}")


def generate(spec: SynthSpec) -> PLC:
    rng = np.random.default_rng(spec.seed)
    n = spec.n_points
    if spec.distribution == "cube":
        pts = rng.uniform(0.0, 1.0, size=(n, 3))
    else:
        pts = np.empty((n, 3))
        have = 0
        while have < n:
            cand = rng.uniform(-1.0, 1.0, size=(2 * (n - have) + 16, 3))
            keep = cand[np.einsum("ij,ij->i", cand, cand) <= 1.0]
            take = min(len(keep), n - have)
            pts[have:have + take] = keep[:take]
            have += take
    cube = spec.distribution == "cube"
    diam = np.sqrt(3.0) if cube else 2.0
    points = [tuple(float(c) for c in p) for p in pts]
    segments, polygons, los, his = [], [], [], []
    for _ in range(int(spec.gamma * n)):
        for _attempt in range(1000):
            axis = int(rng.integers(3))
            center = rng.uniform(0.0, 1.0, size=3) if cube else rng.uniform(-1.0, 1.0, size=3)
            ext = rng.uniform(0.01 * diam, 0.1 * diam, size=2)
            u, v = [k for k in range(3) if k != axis]
            corners = np.tile(center, (4, 1))
            corners[:, u] += np.array([-1, 1, 1, -1]) * (ext[0] / 2)
            corners[:, v] += np.array([-1, -1, 1, 1]) * (ext[1] / 2)
            inside = (np.all(corners >= 0.0) and np.all(corners <= 1.0)) if cube else \
                np.all(np.einsum("ij,ij->i", corners, corners) < 1.0)
            if not inside:
                continue
            lo, hi = corners.min(axis=0), corners.max(axis=0)
            if los and np.any(np.all((lo <= np.array(his)) & (np.array(los) <= hi), axis=1)):
                continue
            b = len(points)
            points.extend(tuple(float(c) for c in q) for q in corners)
            idx = (b, b + 1, b + 2, b + 3)
            segments.extend((min(idx[k], idx[(k + 1) % 4]), max(idx[k], idx[(k + 1) % 4])) for k in range(4))
            polygons.append(idx)
            los.append(lo)
            his.append(hi)
            break
        else:
            raise PlacementFailure("rectangle placement rejected 1000 times")
    return PLC(points=points, segments=segments, polygons=polygons)
