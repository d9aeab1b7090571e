"""Result mesh (drop-in for tetrefine.mesh.Mesh as consumers read it).

Attributes and conventions of /root/reference/pkg/src/tetrefine/mesh.py:9-18,
92-111: ``points[:nv]``, ``vert_origin`` (0 input / 1 Steiner), ``tv`` with the
ghost id -1 in slot 3, ``tn`` packed 4*t+face, ``alive``, ``sub_mask`` /
``seg_mask`` bit sets, ``ratio`` (-1 for ghosts), ``skip_flag``, and the
``subsegments`` {(u,v): sid} / ``subfaces`` {(a,b,c): pid} dictionaries.
The arrays are exported from the GPU once refinement is done.
"""

from __future__ import annotations

import math

import numpy as np

GHOST = -1
FACES = ((1, 2, 3), (0, 3, 2), (0, 1, 3), (0, 2, 1))
EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


class Mesh:
    def __init__(self, arrays: dict, subsegments: dict, subfaces: dict, bbox_diag: float):
        self.points = arrays["points"]
        self.vert_origin = arrays["vert_origin"]
        self.vert_tet = arrays["vert_tet"].astype(np.int64)
        self.tv = arrays["tv"].astype(np.int64)
        self.tn = arrays["tn"].astype(np.int64)
        self.alive = arrays["alive"]
        self.sub_mask = arrays["sub_mask"]
        self.seg_mask = arrays["seg_mask"]
        self.ratio = arrays["ratio"]
        self.skip_flag = arrays["skip_flag"]
        self.nv = len(self.points)
        self.nt = len(self.tv)
        self.subsegments = subsegments
        self.subfaces = subfaces
        self.bbox_diag = bbox_diag
        self.too_close_sq = 1e-24 * bbox_diag * bbox_diag

    def point(self, vid):
        return tuple(float(x) for x in self.points[vid])

    def is_ghost(self, t) -> bool:
        return self.tv[t, 3] == GHOST

    def real_tets(self):
        return [int(t) for t in np.flatnonzero((self.alive[:self.nt] == 1) & (self.tv[:self.nt, 3] != GHOST))]

    def alive_tets(self):
        return [int(t) for t in np.flatnonzero(self.alive[:self.nt] == 1)]

    def n_real_tets(self) -> int:
        return int(np.count_nonzero((self.alive[:self.nt] == 1) & (self.tv[:self.nt, 3] != GHOST)))

    def face_key(self, t, i):
        return tuple(sorted(int(self.tv[t, k]) for k in FACES[i]))

    # -- audits (mesh.py:947-1007), vectorised -----------------------------
    def audit(self, check_delaunay: bool = False):
        """Structural audit: orientation, symmetric neighbours, face pairing,
        mask consistency and constraint presence.  Raises AssertionError."""
        from . import exactnp
        A = np.flatnonzero(self.alive[:self.nt] == 1)
        tv, tn = self.tv[A], self.tn[A]
        ghost = tv[:, 3] == GHOST
        assert np.all((tv[:, :3] >= 0)), "ghost outside slot 3"
        real = A[~ghost]
        if len(real):
            P = self.points
            q = self.tv[real]
            s = exactnp.orient3d_batch(P[q[:, 0]], P[q[:, 1]], P[q[:, 2]], P[q[:, 3]])
            assert np.all(s > 0), f"{int(np.sum(s <= 0))} tets not positively oriented"
        u = tn >> 2
        j = tn & 3
        assert np.all(tn >= 0), "unset neighbour"
        assert np.all(self.alive[u] == 1), "dead neighbour"
        back = self.tn[u, j]
        assert np.all(back == 4 * A[:, None] + np.arange(4)[None, :]), "asymmetric neighbour links"
        fk = np.sort(np.stack([tv[:, list(f)] for f in FACES], axis=1), axis=2)    # (n,4,3)
        keys = fk.reshape(-1, 3)
        # every face key shared by exactly two alive tets
        _, counts = np.unique(keys, axis=0, return_counts=True)
        assert np.all(counts == 2), "face not shared by exactly two tets"
        # masks agree with the dictionaries
        subset = set(self.subfaces)
        for idx in range(len(A)):
            sm = int(self.sub_mask[A[idx]])
            for i in range(4):
                has = tuple(int(x) for x in fk[idx, i]) in subset
                assert bool(sm & (1 << i)) == has, f"sub_mask stale on {A[idx]}:{i}"
        # constraint presence
        keyset = {tuple(int(x) for x in k) for k in keys}
        for key in self.subfaces:
            assert tuple(key) in keyset, f"subface {key} missing"
        edges = set()
        for k in range(6):
            a, b = EDGES[k]
            e = np.sort(tv[:, [a, b]], axis=1)
            edges.update(map(tuple, e[(e >= 0).all(axis=1)].tolist()))
        for key in self.subsegments:
            assert tuple(key) in edges, f"subsegment {key} missing"
        if check_delaunay:
            assert self.delaunay_ok(), "empty-circumsphere violation"

    def delaunay_ok(self) -> bool:
        """Local Delaunay test over every interior face between two real tets
        (equivalent to the global empty-sphere property for a triangulation)."""
        from . import exactnp
        A = np.flatnonzero((self.alive[:self.nt] == 1) & (self.tv[:self.nt, 3] != GHOST))
        P = self.points
        for i in range(4):
            nb = self.tn[A, i]
            u, j = nb >> 2, nb & 3
            ok = self.tv[u, 3] != GHOST
            t = A[ok]
            apex = self.tv[u[ok], j[ok]]
            q = self.tv[t]
            s = exactnp.insphere_batch(P[q[:, 0]], P[q[:, 1]], P[q[:, 2]], P[q[:, 3]], P[apex])
            if np.any(s > 0):
                return False
        return True


def bbox_diag_of(points: np.ndarray) -> float:
    lo, hi = points.min(axis=0), points.max(axis=0)
    return math.dist(tuple(lo), tuple(hi))
