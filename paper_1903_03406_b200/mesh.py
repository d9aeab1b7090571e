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

from dataclasses import dataclass

GHOST = -1
FACES = ((1, 2, 3), (0, 3, 2), (0, 1, 3), (0, 2, 1))
EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


@dataclass(frozen=True)
class ElementRef:
    """Result of a location query (mesh.py:40-50 of the reference)."""
    kind: str
    index: int


OUTSIDE = ElementRef("outside", -1)


def _o3d(a, b, c, d) -> int:
    from . import exactnp
    return int(exactnp.orient3d_batch(np.asarray([a]), np.asarray([b]), np.asarray([c]), np.asarray([d]))[0])


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

    def face_vertices(self, t, i):
        f = FACES[i]
        return (int(self.tv[t, f[0]]), int(self.tv[t, f[1]]), int(self.tv[t, f[2]]))

    def neighbor(self, t, i):
        """(tet, face) across face i of tet t."""
        x = int(self.tn[t, i])
        return x >> 2, x & 3

    # -- adjacency queries (mesh.py:236-293) -------------------------------
    def tets_around_vertex(self, v):
        """All alive tets containing vertex v (DFS from vert_tet; like the
        reference, a stale vert_tet entry is repaired as a side effect)."""
        start = int(self.vert_tet[v])
        if start < 0 or start >= self.nt or not self.alive[start] or v not in self.tv[start]:
            hit = np.flatnonzero((self.alive[:self.nt] == 1) & np.any(self.tv[:self.nt] == v, axis=1))
            if len(hit) == 0:
                return []
            start = int(hit[0])
            self.vert_tet[v] = start
        out = [start]
        seen = {start}
        stack = [start]
        while stack:
            t = stack.pop()
            local = list(self.tv[t]).index(v)
            for i in range(4):
                if i == local:
                    continue
                u = int(self.tn[t, i]) >> 2
                if u >= 0 and u not in seen and self.alive[u]:
                    seen.add(u)
                    out.append(u)
                    stack.append(u)
        return out

    def edge_exists(self, u, v) -> bool:
        return any(v in self.tv[t] for t in self.tets_around_vertex(u))

    def tets_around_edge(self, u, v):
        return [t for t in self.tets_around_vertex(u) if v in self.tv[t]]

    def find_tet_with_face(self, key):
        """(t, i) of an alive tet with the sorted vertex triple as a face, or (-1, -1)."""
        key = tuple(int(k) for k in key)
        for t in self.tets_around_vertex(key[0]):
            tvs = [int(x) for x in self.tv[t]]
            if key[1] in tvs and key[2] in tvs:
                for i in range(4):
                    if self.face_key(t, i) == key:
                        return t, i
        return -1, -1

    def edge_link_vertices(self, u, v):
        """Vertices opposite the edge (u, v) in its tets, ghosts excluded."""
        out = set()
        for t in self.tets_around_edge(u, v):
            for w in self.tv[t]:
                w = int(w)
                if w not in (u, v, GHOST):
                    out.add(w)
        return out

    # -- location (mesh.py:297-391) -----------------------------------------
    def locate(self, p, hint=None):
        """ElementRef("tet", t) with t the lowest-index alive real tet
        containing p, or OUTSIDE (exact predicates)."""
        t = self._walk(p, hint)
        if self.is_ghost(t):
            return OUTSIDE
        return ElementRef("tet", self._lowest_containing(p, t))

    def _hint_tet(self, hint):
        if isinstance(hint, ElementRef):
            hint = hint.index if hint.kind == "tet" else None
        if hint is not None and 0 <= hint < self.nt and self.alive[hint] and not self.is_ghost(hint):
            return int(hint)
        real = np.flatnonzero((self.alive[:self.nt] == 1) & (self.tv[:self.nt, 3] != GHOST))
        if len(real) == 0:
            from .errors import CavityNotStarShaped
            raise CavityNotStarShaped("mesh has no alive real tets")
        return int(real[0])

    def _walk(self, p, hint=None):
        """Stochastic remembering walk; a real tet containing p or a ghost
        tet whose outer half-space holds p (exhaustive scan as a last resort)."""
        p = tuple(float(x) for x in p)
        t = self._hint_tet(hint)
        max_steps = int(10 * max(1.0, self.nt) ** (1.0 / 3.0)) + 32
        prev = -1
        for step in range(1, max_steps + 1):
            if self.is_ghost(t):
                return t
            moved = False
            for k in range(4):
                i = (k + step) & 3
                u = int(self.tn[t, i]) >> 2
                if u == prev:
                    continue
                fv = self.face_vertices(t, i)
                if _o3d(self.points[fv[0]], self.points[fv[1]], self.points[fv[2]], p) > 0:
                    prev, t, moved = t, u, True
                    break
            if not moved:
                return t
        for t in self.real_tets():
            if all(_o3d(*(self.points[v] for v in self.face_vertices(t, i)), p) <= 0 for i in range(4)):
                return t
        for t in self.alive_tets():
            if self.is_ghost(t) and _o3d(*(self.points[self.tv[t, k]] for k in range(3)), p) > 0:
                return t
        from .errors import CavityNotStarShaped
        raise CavityNotStarShaped("walk failed to locate point")

    def _lowest_containing(self, p, t):
        found = {t}
        stack = [t]
        while stack:
            cur = stack.pop()
            for i in range(4):
                fv = self.face_vertices(cur, i)
                if _o3d(self.points[fv[0]], self.points[fv[1]], self.points[fv[2]], p) == 0:
                    u = int(self.tn[cur, i]) >> 2
                    if u >= 0 and self.alive[u] and not self.is_ghost(u) and u not in found:
                        if all(_o3d(*(self.points[v] for v in self.face_vertices(u, j)), p) <= 0 for j in range(4)):
                            found.add(u)
                            stack.append(u)
        return min(found)

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
