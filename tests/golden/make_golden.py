"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
(/root/reference/pkg/src, read-only) in this container.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed as
small .npz files:
  * predicates.npz -- orient2d/incircle2d/orient3d/insphere/incircle3d and
    encroachment signs on random and near-degenerate inputs, plus
    circumsphere/circumcircle constructions (bit patterns);
  * refine_<case>.npz -- final point array, origins, constraint sets, a
    hash of the real-tet vertex tuples, per-round statistics and skip list of
    ``tetrefine.refine`` on small seeded PLCs built by
    paper_1903_03406_b200.synth.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import tetrefine  # noqa: E402
from tetrefine import geometry as G  # noqa: E402
from tetrefine import predicates as P  # noqa: E402


from tests.golden.cases import CASES, tet_hash  # noqa: E402


def predicate_corpus(rng, n):
    """Random points plus perturbations of exactly degenerate configurations."""
    out = {}
    # orient3d: random, exact coplanar (integer grid), and 1e-12 perturbed
    r = rng.uniform(-1, 1, (n, 4, 3))
    cop = rng.integers(-4, 5, (n, 4, 3)).astype(np.float64)
    cop[:, :, 2] = 0.5 * cop[:, :, 0] - 0.25 * cop[:, :, 1] + 1.0   # coplanar
    pert = cop.copy()
    pert[:, 3, :] += rng.normal(size=(n, 3)) * 1e-12
    tiny = cop * 1e-3 + rng.normal(size=(n, 4, 3)) * 1e-19
    out["o3d_in"] = np.concatenate([r, cop, pert, tiny]).reshape(-1, 12)
    # insphere: random, cospherical (points on the unit sphere from Pythagorean
    # quadruples), perturbed
    r5 = rng.uniform(-1, 1, (n, 5, 3))
    quads = np.array([(1, 2, 2, 3), (2, 3, 6, 7), (1, 4, 8, 9), (4, 4, 7, 9), (2, 6, 9, 11), (6, 6, 7, 11)],
                     dtype=np.float64)
    sph = np.zeros((n, 5, 3))
    for i in range(n):
        for k in range(5):
            a, b, c, d = quads[rng.integers(len(quads))]
            s = rng.choice([-1.0, 1.0], 3)
            perm = rng.permutation(3)
            v = np.array([a, b, c])[perm] * s / d
            sph[i, k] = v
    # orient positively (swap a,b when negative)
    for i in range(n):
        if P.orient3d(*[tuple(x) for x in sph[i, :4]]) < 0:
            sph[i, [0, 1]] = sph[i, [1, 0]]
        if P.orient3d(*[tuple(x) for x in r5[i, :4]]) < 0:
            r5[i, [0, 1]] = r5[i, [1, 0]]
    sp = sph.copy()
    sp[:, 4, :] *= 1.0 + rng.normal(size=(n, 1)) * 1e-14
    out["isp_in"] = np.concatenate([r5, sph, sp]).reshape(-1, 15)
    # orient2d / incircle2d
    r3 = rng.uniform(-1, 1, (n, 3, 2))
    col = rng.integers(-8, 9, (n, 3, 2)).astype(np.float64)
    col[:, 2] = col[:, 0] + (col[:, 1] - col[:, 0]) * 0.5
    out["o2d_in"] = np.concatenate([r3, col, col + rng.normal(size=(n, 3, 2)) * 1e-15]).reshape(-1, 6)
    r4 = rng.uniform(-1, 1, (n, 4, 2))
    circ = np.zeros((n, 4, 2))
    pyth = [(3, 4, 5), (5, 12, 13), (8, 15, 17), (7, 24, 25)]
    for i in range(n):
        for k in range(4):
            a, b, c = pyth[rng.integers(4)]
            s = rng.choice([-1.0, 1.0], 2)
            circ[i, k] = (np.array([a, b]) if rng.integers(2) else np.array([b, a])) * s / c
        if P.orient2d(tuple(circ[i, 0]), tuple(circ[i, 1]), tuple(circ[i, 2])) < 0:
            circ[i, [0, 1]] = circ[i, [1, 0]]
    out["icc_in"] = np.concatenate([r4, circ]).reshape(-1, 8)
    # incircle3d: coplanar quadruples in random planes (exactly representable:
    # z = x/2 - y/4) and axis planes
    q = rng.integers(-6, 7, (n, 4, 3)).astype(np.float64)
    q[:, :, 2] = 0.5 * q[:, :, 0] - 0.25 * q[:, :, 1]
    out["inc3_in"] = q.reshape(-1, 12)
    # encroachment: segment balls and equatorial balls, with boundary cases
    seg = rng.uniform(-1, 1, (n, 3, 3))
    segb = np.zeros((n, 3, 3))
    segb[:, 0] = (0, 0, 0)
    segb[:, 1] = (2, 0, 0)
    segb[:, 2] = np.stack([np.ones(n), np.cos(np.linspace(0, 6, n)).round(0), np.zeros(n)], axis=1)
    out["eseg_in"] = np.concatenate([seg, segb]).reshape(-1, 9)
    tri = rng.uniform(-1, 1, (n, 4, 3))
    trib = np.zeros((n, 4, 3))
    trib[:, 1] = (2, 0, 0)
    trib[:, 2] = (0, 2, 0)
    trib[:, 3] = np.stack([np.ones(n), np.ones(n), np.where(np.arange(n) % 2 == 0, np.sqrt(2.0), 1.0)], axis=1)
    out["eface_in"] = np.concatenate([tri, trib]).reshape(-1, 12)
    return out


def eval_predicates(c):
    res = {}
    res["o3d"] = np.array([P.orient3d(*[tuple(x) for x in row.reshape(4, 3)]) for row in c["o3d_in"]], np.int8)
    res["isp"] = np.array([P.insphere(*[tuple(x) for x in row.reshape(5, 3)]) for row in c["isp_in"]], np.int8)
    res["o2d"] = np.array([P.orient2d(*[tuple(x) for x in row.reshape(3, 2)]) for row in c["o2d_in"]], np.int8)
    res["icc"] = np.array([P.incircle2d(*[tuple(x) for x in row.reshape(4, 2)]) for row in c["icc_in"]], np.int8)
    inc = []
    for row in c["inc3_in"]:
        try:
            inc.append(P.incircle3d(*[tuple(x) for x in row.reshape(4, 3)]))
        except ValueError:
            inc.append(99)
    res["inc3"] = np.array(inc, np.int8)
    res["eseg"] = np.array([G.encroaches_segment((tuple(r[0:3]), tuple(r[3:6])), tuple(r[6:9]))
                            for r in c["eseg_in"]], np.int8)
    ef = []
    for r in c["eface_in"]:
        try:
            ef.append(int(G.encroaches_face((tuple(r[0:3]), tuple(r[3:6]), tuple(r[6:9])), tuple(r[9:12]))))
        except Exception:
            ef.append(99)
    res["eface"] = np.array(ef, np.int8)
    cs = []
    for row in c["o3d_in"][: len(c["o3d_in"]) // 4]:
        try:
            s = G.circumsphere_tet(*[tuple(x) for x in row.reshape(4, 3)])
            cs.append(list(s.center) + [s.radius_sq])
        except Exception:
            cs.append([np.nan] * 4)
    res["csph"] = np.array(cs)
    cc = []
    for row in c["o3d_in"][: len(c["o3d_in"]) // 4]:
        try:
            s = G.circumcircle_tri(*[tuple(x) for x in row.reshape(4, 3)[:3]])
            cc.append(list(s.center) + [s.radius_sq])
        except Exception:
            cc.append([np.nan] * 4)
    res["ccir"] = np.array(cc)
    return res


def main(which=None):
    rng = np.random.default_rng(1234)
    corpus = predicate_corpus(rng, 500)
    res = eval_predicates(corpus)
    np.savez_compressed(os.path.join(HERE, "predicates.npz"), **corpus, **{"out_" + k: v for k, v in res.items()})
    print("predicates.npz", {k: len(v) for k, v in res.items()})
    for name, (build, B) in CASES.items():
        if which and name not in which:
            continue
        plc = build()
        rplc = tetrefine.PLC(points=plc.points, segments=plc.segments, polygons=plc.polygons)
        mesh, rep = tetrefine.refine(rplc, tetrefine.RefineConfig(B=B))
        real = [mesh.tv[t] for t in mesh.real_tets()]
        per_round = np.array([[r["round"], {"segments": 0, "faces": 1, "tets": 2}[r["phase"]], r["candidates"],
                               r["accepted"], r["blasted"], r["failed"], r["inserted"], r["pending_segments"],
                               r["pending_faces"]] for r in rep.per_round], dtype=np.int64).reshape(-1, 9)
        segs = np.array(sorted((u, v, s) for (u, v), s in mesh.subsegments.items()), dtype=np.int32).reshape(-1, 3)
        faces = np.array(sorted((a, b, c, p) for (a, b, c), p in mesh.subfaces.items()), dtype=np.int32).reshape(-1, 4)
        np.savez_compressed(
            os.path.join(HERE, f"refine_{name}.npz"),
            B=B, points=mesh.points[:mesh.nv].copy(), vert_origin=mesh.vert_origin[:mesh.nv].copy(),
            subsegments=segs, subfaces=faces, tet_hash=np.array(tet_hash(real)), n_real_tets=len(real),
            per_round=per_round, steiner=rep.steiner_points, tet_count=rep.tet_count,
            bad_tet_count=rep.bad_tet_count, hist=np.array(rep.dihedral_histogram),
            skipped=np.array(json.dumps(rep.skipped)))
        print(name, "nv", mesh.nv, "steiner", rep.steiner_points, "tets", rep.tet_count, "rounds",
              len(rep.per_round), "skipped", len(rep.skipped))


if __name__ == "__main__":
    main(sys.argv[1:] or None)
