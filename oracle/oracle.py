"""TEST INFRASTRUCTURE ONLY: ctypes binding of the CPU oracle (liboracle.so).

Imported by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) as the checker / CPU baseline -- never by the product
package.  The oracle is a sequential C++ restatement of the reference round
driver (/root/reference/pkg/src/tetrefine/refine.py) whose outputs are pinned
bit-for-bit against the reference's own outputs in tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build(force: bool = False) -> str:
    path = os.path.join(_HERE, "liboracle.so")
    if force or not os.path.exists(path):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return path


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        vp, i32, f64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        L.or_refine.restype = vp
        L.or_refine.argtypes = [vp, i32, i32, vp, i32, vp, vp, i32, vp, f64, i32, ctypes.c_ulonglong]
        for name in ("or_free", "or_counts", "or_mesh", "or_constraints", "or_rounds", "or_skipped", "or_times",
                     "or_status"):
            getattr(L, name).restype = None if name != "or_status" else i32
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


PHASES = {0: "segments", 1: "faces", 2: "tets"}
REASONS = {0: "degenerate", 1: "short_edge", 2: "too_close", 3: "cavity_not_star_shaped"}
KINDS = {0: "subsegment", 1: "subface", 2: "tet"}


def refine_prepared(prep, B: float, max_rounds: int = 500, seed: int = 0) -> dict:
    """Run the oracle on a ``paper_1903_03406_b200.prepare.Prepared``."""
    L = lib()
    t0 = time.perf_counter()
    h = L.or_refine(_p(prep.points), len(prep.points), prep.n_input, _p(prep.segments), len(prep.segments),
                    _p(prep.poly_off), _p(prep.poly_idx), len(prep.poly_off) - 1, _p(prep.order),
                    float(B), int(max_rounds), ctypes.c_ulonglong(seed & 0xFFFFFFFFFFFFFFFF))
    wall = time.perf_counter() - t0
    try:
        buf = ctypes.create_string_buffer(256)
        st = L.or_status(h, buf, 256)
        if st != 0:
            raise RuntimeError("oracle failed: " + buf.value.decode())
        cnt = np.zeros(9, dtype=np.int64)
        L.or_counts(h, _p(cnt))
        nv, nt, ns, nf, nr, nsk = (int(x) for x in cnt[:6])
        out = dict(nv=nv, nt=nt, exact_o3d=int(cnt[6]), exact_isp=int(cnt[7]), region_calls=int(cnt[8]))
        pts = np.zeros((nv, 3)); origin = np.zeros(nv, np.uint8); vt = np.zeros(nv, np.int32)
        tv = np.zeros((nt, 4), np.int32); tn = np.zeros((nt, 4), np.int64); alive = np.zeros(nt, np.uint8)
        sm = np.zeros(nt, np.uint8); em = np.zeros(nt, np.uint8); ratio = np.zeros(nt); skip = np.zeros(nt, np.uint8)
        L.or_mesh(h, _p(pts), _p(origin), _p(vt), _p(tv), _p(tn), _p(alive), _p(sm), _p(em), _p(ratio), _p(skip))
        segs = np.zeros((ns, 3), np.int32); faces = np.zeros((nf, 4), np.int32)
        L.or_constraints(h, _p(segs), _p(faces))
        rows = np.zeros((nr, 9), np.int64); times = np.zeros(nr)
        L.or_rounds(h, _p(rows), _p(times))
        sk = np.zeros((nsk, 7), np.int32)
        L.or_skipped(h, _p(sk))
        tt = np.zeros(2)
        L.or_times(h, _p(tt))
        out.update(points=pts, vert_origin=origin, vert_tet=vt, tv=tv, tn=tn, alive=alive, sub_mask=sm, seg_mask=em,
                   ratio=ratio, skip_flag=skip, subsegments=segs, subfaces=faces, wall=wall, setup_time=tt[0],
                   total_time=tt[1])
        out["per_round"] = [dict(round=int(r[0]), phase=PHASES[int(r[1])], candidates=int(r[2]), accepted=int(r[3]),
                                 blasted=int(r[4]), failed=int(r[5]), inserted=int(r[6]),
                                 pending_segments=int(r[7]), pending_faces=int(r[8]), time=float(t))
                            for r, t in zip(rows, times)]
        out["skipped"] = [dict(kind=KINDS[int(r[0])], vertices=[int(x) for x in r[3:3 + r[2]]], reason=REASONS[int(r[1])])
                          for r in sk]
        return out
    finally:
        L.or_free(h)


def refine(plc, B: float = 2.0, max_rounds: int = 500, seed: int = 0) -> dict:
    sys.path.insert(0, os.path.dirname(_HERE))
    from paper_1903_03406_b200.prepare import prepare

    prep = prepare(plc, seed=seed)
    out = refine_prepared(prep, B, max_rounds, seed)
    out["prepare_s"] = prep.setup_s
    return out


def batch(name: str, arr: np.ndarray, out_dtype=np.int8, width: int = 1) -> np.ndarray:
    """Batched predicate / construction entry points (or_orient3d, ...)."""
    L = lib()
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    n = arr.shape[0]
    out = np.zeros((n, width) if width > 1 else n, dtype=out_dtype)
    getattr(L, name)(_p(arr), ctypes.c_int(n), _p(out))
    return out
