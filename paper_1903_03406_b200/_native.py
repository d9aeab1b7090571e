"""ctypes binding of libgqm3d.so (include/gqm3d.h).

There is no CPU fallback: if the library or a CUDA device is missing every
entry point raises ``NativeError`` / ``OSError``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class GqConfig(ctypes.Structure):
    _fields_ = [("B", ctypes.c_double), ("max_rounds", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("seed", ctypes.c_uint64)]


class GqCounts(ctypes.Structure):
    _fields_ = [("nv", ctypes.c_int64), ("nt", ctypes.c_int64), ("n_subsegments", ctypes.c_int64),
                ("n_subfaces", ctypes.c_int64), ("n_rounds", ctypes.c_int64), ("n_skipped", ctypes.c_int64),
                ("n_real_tets", ctypes.c_int64), ("steiner_points", ctypes.c_int64),
                ("input_points", ctypes.c_int64), ("exact_calls", ctypes.c_int64 * 4),
                ("device_ms", ctypes.c_double), ("init_ms", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64), ("region_calls", ctypes.c_int64),
                ("bytes_alg", ctypes.c_int64), ("region_ms", ctypes.c_double),
                ("n_cand", ctypes.c_int64), ("t_tested", ctypes.c_int64), ("k_claims", ctypes.c_int64),
                ("t_created", ctypes.c_int64), ("t_deleted", ctypes.c_int64), ("bytes_refine", ctypes.c_int64)]


EXPORTS = ("gq_create", "gq_destroy", "gq_last_error", "gq_refine", "gq_export_mesh", "gq_export_constraints",
           "gq_export_rounds", "gq_export_skipped", "gq_quality", "gq_batch", "gq_write_mesh", "gq_certify_pairs",
           "gq_probe_fp64")


def lib_path() -> str:
    return os.environ.get("GQM3D_LIB", os.path.join(_HERE, "libgqm3d.so"))


def lib():
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            raise OSError(f"libgqm3d.so not built ({path}); run paper_1903_03406_b200.build.build()")
        L = ctypes.CDLL(path)
        vp, i32 = ctypes.c_void_p, ctypes.c_int32
        L.gq_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        L.gq_destroy.argtypes = [vp]
        L.gq_last_error.argtypes = [vp]
        L.gq_last_error.restype = ctypes.c_char_p
        L.gq_refine.argtypes = [vp, vp, i32, i32, vp, i32, vp, vp, i32, vp, vp, ctypes.POINTER(GqConfig),
                                ctypes.POINTER(GqCounts)]
        L.gq_export_mesh.argtypes = [vp] * 11
        L.gq_export_constraints.argtypes = [vp, vp, vp]
        L.gq_export_rounds.argtypes = [vp, vp, vp]
        L.gq_export_skipped.argtypes = [vp, vp]
        L.gq_quality.argtypes = [vp, ctypes.c_double, vp, vp, vp, ctypes.c_int64, vp]
        L.gq_batch.argtypes = [ctypes.c_int, vp, i32, i32, vp, vp]
        L.gq_write_mesh.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, vp, vp, i32, vp, vp, i32, vp, i32]
        if hasattr(L, "gq_probe_fp64"):        # (an older library in GQM3D_LIB may lack the newer entry points)
            L.gq_probe_fp64.argtypes = [ctypes.c_int, vp]
        if hasattr(L, "gq_certify_pairs"):
            L.gq_certify_pairs.argtypes = [ctypes.c_int, vp, i32, vp, i32, vp, i32, vp, vp, ctypes.c_int64, vp]
        for name in EXPORTS:
            if name not in ("gq_last_error",) and hasattr(L, name):
                getattr(L, name).restype = ctypes.c_int
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Context:
    """One GPU-resident mesh context (one refine at a time)."""

    def __init__(self, device: int = 0):
        self._L = lib()
        self._h = ctypes.c_void_p()
        st = self._L.gq_create(int(device), ctypes.byref(self._h))
        if st != 0:
            msg = self._L.gq_last_error(self._h).decode()
            self._L.gq_destroy(self._h)
            self._h = None
            raise NativeError(st, msg)

    def _check(self, st):
        if st != 0:
            raise NativeError(st, self._L.gq_last_error(self._h).decode())

    def close(self):
        if self._h:
            self._L.gq_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def refine(self, prep, keep: np.ndarray, B: float, max_rounds: int, seed: int, verbose: bool = False,
               blast: bool = False) -> GqCounts:
        cfg = GqConfig(float(B), int(max_rounds), (1 if verbose else 0) | (2 if blast else 0),
                       int(seed) & 0xFFFFFFFFFFFFFFFF)
        cnt = GqCounts()
        keep = np.ascontiguousarray(keep, dtype=np.int32)
        self._check(self._L.gq_refine(self._h, _p(prep.points), len(prep.points), prep.n_input, _p(prep.segments),
                                      len(prep.segments), _p(prep.poly_off), _p(prep.poly_idx),
                                      len(prep.poly_off) - 1, _p(keep), _p(prep.order), ctypes.byref(cfg),
                                      ctypes.byref(cnt)))
        return cnt

    def export_mesh(self, cnt: GqCounts) -> dict:
        nv, nt = int(cnt.nv), int(cnt.nt)
        out = dict(points=np.zeros((nv, 3)), vert_origin=np.zeros(nv, np.uint8), vert_tet=np.zeros(nv, np.int32),
                   tv=np.zeros((nt, 4), np.int32), tn=np.zeros((nt, 4), np.int32), alive=np.zeros(nt, np.uint8),
                   sub_mask=np.zeros(nt, np.uint8), seg_mask=np.zeros(nt, np.uint8), ratio=np.zeros(nt),
                   skip_flag=np.zeros(nt, np.uint8))
        self._check(self._L.gq_export_mesh(self._h, *(_p(out[k]) for k in (
            "points", "vert_origin", "vert_tet", "tv", "tn", "alive", "sub_mask", "seg_mask", "ratio", "skip_flag"))))
        return out

    def export_constraints(self, cnt: GqCounts):
        s = np.zeros((int(cnt.n_subsegments), 3), np.int32)
        f = np.zeros((int(cnt.n_subfaces), 4), np.int32)
        self._check(self._L.gq_export_constraints(self._h, _p(s), _p(f)))
        return s, f

    def export_rounds(self, cnt: GqCounts):
        rows = np.zeros((int(cnt.n_rounds), 9), np.int64)
        secs = np.zeros(int(cnt.n_rounds))
        self._check(self._L.gq_export_rounds(self._h, _p(rows), _p(secs)))
        return rows, secs

    def export_skipped(self, cnt: GqCounts):
        rows = np.zeros((int(cnt.n_skipped), 7), np.int32)
        self._check(self._L.gq_export_skipped(self._h, _p(rows)))
        return rows

    def quality(self, B: float, edge_cap: int = 1 << 22):
        """(bad count, device histogram, tets whose dihedral angles sit on a
        bin edge -- to be binned by the caller with the reference's formula)."""
        bad = np.zeros(1, np.int64)
        hist = np.zeros(36, np.int64)
        edges = np.zeros(edge_cap, np.int32)
        ne = np.zeros(1, np.int64)
        self._check(self._L.gq_quality(self._h, float(B), _p(bad), _p(hist), _p(edges), int(edge_cap), _p(ne)))
        return int(bad[0]), hist, edges[:int(ne[0])]


_BATCH = {"orient3d": (0, 12), "insphere": (1, 15), "orient2d": (2, 6), "incircle2d": (3, 8),
          "incircle3d": (4, 12), "encroaches_segment": (5, 9), "encroaches_face": (6, 12),
          "circumsphere_tet": (7, 12), "circumcircle_tri": (8, 9)}


def batch(name: str, arr: np.ndarray) -> np.ndarray:
    """Evaluate a predicate / construction on the GPU for every row of arr."""
    which, width = _BATCH[name]
    arr = np.ascontiguousarray(arr, dtype=np.float64).reshape(-1, width)
    n = len(arr)
    if which >= 7:
        out = np.zeros((n, 4))
        st = lib().gq_batch(which, _p(arr), n, width, None, _p(out))
    else:
        out = np.zeros(n, np.int8)
        st = lib().gq_batch(which, _p(arr), n, width, _p(out), None)
    if st != 0:
        raise NativeError(st, "gq_batch failed")
    return out


def certify_pairs(points: np.ndarray, segments: np.ndarray, triangles: np.ndarray, device: int = 0,
                  cap: int = 1 << 20):
    """Feature-pair certification of a PLC on the device (include/gqm3d.h
    gq_certify_pairs).  Returns (status, undecided pairs (k, 2))."""
    P = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    S = np.ascontiguousarray(segments, dtype=np.int32).reshape(-1, 2)
    T = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
    st = np.zeros(1, np.int32)
    npairs = np.zeros(1, np.int64)
    pairs = np.zeros((cap, 2), np.int32)
    rc = lib().gq_certify_pairs(int(device), _p(P), len(P), _p(S), len(S), _p(T), len(T), _p(st), _p(pairs),
                                int(cap), _p(npairs))
    if rc != 0:
        raise NativeError(rc, "gq_certify_pairs failed")
    return int(st[0]), pairs[:int(npairs[0])]


def probe_fp64(device: int = 0) -> float:
    """Measured FP64 FMA peak of the device in TFLOP/s (gq_probe_fp64)."""
    out = np.zeros(1)
    rc = lib().gq_probe_fp64(int(device), _p(out))
    if rc != 0:
        raise NativeError(rc, "gq_probe_fp64 failed")
    return float(out[0])
