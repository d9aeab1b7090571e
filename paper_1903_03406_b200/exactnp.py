"""Vectorised exact orient3d / insphere for host-side audits.

Float filter with the reference's error bounds
(/root/reference/pkg/src/tetrefine/predicates.py:31-34, 169-283); entries the
filter cannot certify are decided exactly on Python integers (frexp scaling,
predicates.py:55-126).  Used only by ``Mesh.audit`` / ``delaunay_ok``.
"""

from __future__ import annotations

import math

import numpy as np

_EPS = 2.0 ** -53
_O3D = (7.0 + 56.0 * _EPS) * _EPS
_ISP = (16.0 + 224.0 * _EPS) * _EPS


def _ints(xs):
    fr = [math.frexp(float(x)) for x in xs]
    emin = min(e for _, e in fr)
    return [int(m * (1 << 53)) << (e - emin) for m, e in fr]


def _o3d_exact(a, b, c, d):
    v = _ints(list(a) + list(b) + list(c) + list(d))
    u = [v[3 + k] - v[k] for k in range(3)]
    w1 = [v[6 + k] - v[k] for k in range(3)]
    w2 = [v[9 + k] - v[k] for k in range(3)]
    det = (u[0] * (w1[1] * w2[2] - w1[2] * w2[1]) - u[1] * (w1[0] * w2[2] - w1[2] * w2[0])
           + u[2] * (w1[0] * w2[1] - w1[1] * w2[0]))
    return (det > 0) - (det < 0)


def _isp_exact(a, b, c, d, e):
    v = _ints(list(a) + list(b) + list(c) + list(d) + list(e))
    rows = []
    for k in range(4):
        px, py, pz = v[3 * k] - v[12], v[3 * k + 1] - v[13], v[3 * k + 2] - v[14]
        rows.append((px, py, pz, px * px + py * py + pz * pz))

    def det3(r0, r1, r2):
        return (r0[0] * (r1[1] * r2[2] - r1[2] * r2[1]) - r0[1] * (r1[0] * r2[2] - r1[2] * r2[0])
                + r0[2] * (r1[0] * r2[1] - r1[1] * r2[0]))

    r0, r1, r2, r3 = rows
    det = -r0[3] * det3(r1, r2, r3) + r1[3] * det3(r0, r2, r3) - r2[3] * det3(r0, r1, r3) + r3[3] * det3(r0, r1, r2)
    return -((det > 0) - (det < 0))


def orient3d_batch(a, b, c, d):
    ad, bd, cd = a - d, b - d, c - d
    t1 = bd[:, 0] * cd[:, 1]; t2 = cd[:, 0] * bd[:, 1]
    t3 = cd[:, 0] * ad[:, 1]; t4 = ad[:, 0] * cd[:, 1]
    t5 = ad[:, 0] * bd[:, 1]; t6 = bd[:, 0] * ad[:, 1]
    det = ad[:, 2] * (t1 - t2) + bd[:, 2] * (t3 - t4) + cd[:, 2] * (t5 - t6)
    perm = (np.abs(ad[:, 2]) * (np.abs(t1) + np.abs(t2)) + np.abs(bd[:, 2]) * (np.abs(t3) + np.abs(t4))
            + np.abs(cd[:, 2]) * (np.abs(t5) + np.abs(t6)))
    out = -np.sign(det).astype(np.int64)
    unsure = np.flatnonzero(~(np.abs(det) > _O3D * perm))
    for i in unsure:
        out[i] = _o3d_exact(a[i], b[i], c[i], d[i])
    return out


def insphere_batch(a, b, c, d, e):
    A, Bm, C, Dm = a - e, b - e, c - e, d - e
    lift = [np.einsum("ij,ij->i", X, X) for X in (A, Bm, C, Dm)]

    def det3(X, Y, Z):
        return (X[:, 0] * (Y[:, 1] * Z[:, 2] - Y[:, 2] * Z[:, 1]) - X[:, 1] * (Y[:, 0] * Z[:, 2] - Y[:, 2] * Z[:, 0])
                + X[:, 2] * (Y[:, 0] * Z[:, 1] - Y[:, 1] * Z[:, 0]))

    det = (-lift[0] * det3(Bm, C, Dm) + lift[1] * det3(A, C, Dm) - lift[2] * det3(A, Bm, Dm)
           + lift[3] * det3(A, Bm, C))
    mag = sum(l * (np.abs(X).sum(axis=1) ** 3) for l, X in zip(lift, (A, Bm, C, Dm))) + 1e-300
    out = -np.sign(det).astype(np.int64)
    unsure = np.flatnonzero(~(np.abs(det) > 64 * _ISP * mag))
    for i in unsure:
        out[i] = _isp_exact(a[i], b[i], c[i], d[i], e[i])
    return out
