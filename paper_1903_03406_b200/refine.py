"""``refine(plc, cfg)`` -- the drop-in entry point (refine.py:928-933).

Host work is the reference's own setup (validation, box closure, insertion
order; refine.py:523-531, mesh.py:873-880).  Everything from the initial
Delaunay tetrahedralization to the final verification scan runs on the GPU
through libgqm3d.so (include/gqm3d.h); the result is exported once into a
``Mesh`` and a ``QualityReport``.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import _native
from .config import RefineConfig
from .mesh import Mesh, bbox_diag_of
from .plc import PLC
from .prepare import facet_keep, prepare
from .stats import QualityReport

_PHASES = {0: "segments", 1: "faces", 2: "tets"}
_KINDS = {0: "subsegment", 1: "subface", 2: "tet"}
_REASONS = {0: "degenerate", 1: "short_edge", 2: "too_close", 3: "cavity_not_star_shaped"}
_CTX = {}


def _context(device: int) -> _native.Context:
    ctx = _CTX.get(device)
    if ctx is None:
        ctx = _CTX[device] = _native.Context(device)
    return ctx


def default_device() -> int:
    return int(os.environ.get("GQM3D_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def refine(plc: PLC, cfg: RefineConfig = None, device: int = None, context: _native.Context = None):
    """Refine ``plc`` into a conforming tetrahedral mesh whose tets have
    radius-edge ratio <= cfg.B (up to the reference's skip rules).
    Returns ``(Mesh, QualityReport)``.  ``cfg`` may also be a bare float B."""
    if cfg is None:
        cfg = RefineConfig()
    elif isinstance(cfg, (int, float)):
        cfg = RefineConfig(B=float(cfg))
    t0 = time.perf_counter()
    prep = prepare(plc, seed=cfg.seed)
    keep = facet_keep(prep.plc)
    t_prep = time.perf_counter() - t0
    ctx = context if context is not None else _context(default_device() if device is None else device)
    cnt = ctx.refine(prep, keep, cfg.B, cfg.max_rounds, cfg.seed, cfg.verbose, blast=cfg.filter == "blast")
    t_dev = time.perf_counter() - t0 - t_prep
    t1 = time.perf_counter()
    arrays = ctx.export_mesh(cnt)
    segs, faces = ctx.export_constraints(cnt)
    rows, secs = ctx.export_rounds(cnt)
    sk = ctx.export_skipped(cnt)
    bad, hist, edge_tets = ctx.quality(cfg.B)
    mesh = Mesh(arrays, {(int(u), int(v)): int(s) for u, v, s in segs},
                {(int(a), int(b), int(c)): int(p) for a, b, c, p in faces}, bbox_diag_of(prep.points))
    rep = QualityReport()
    org = arrays["vert_origin"]
    rep.input_points = int(np.count_nonzero(org == 0))
    rep.steiner_points = int(np.count_nonzero(org == 1))
    rep.tet_count = mesh.n_real_tets()
    rep.bad_tet_count = bad
    if len(edge_tets):   # bin-edge angles: the reference's own numpy expression (stats.py:64-86)
        from .stats import dihedral_histogram_of
        hist = hist + dihedral_histogram_of(mesh.points, mesh.tv[edge_tets])
    rep.dihedral_histogram = [int(x) for x in hist]
    rep.skipped = [{"kind": _KINDS[int(r[0])], "vertices": [int(x) for x in r[3:3 + r[2]]],
                    "reason": _REASONS[int(r[1])]} for r in sk]
    rep.per_round = [{"round": int(r[0]), "phase": _PHASES[int(r[1])], "candidates": int(r[2]),
                      "accepted": int(r[3]), "blasted": int(r[4]), "failed": int(r[5]), "inserted": int(r[6]),
                      "pending_segments": int(r[7]), "pending_faces": int(r[8]), "workers": cfg.workers,
                      "time": float(t)} for r, t in zip(rows, secs)]
    t_exp = time.perf_counter() - t1
    rep.total_time = time.perf_counter() - t0
    rep.device = {"device_ms": cnt.device_ms, "init_ms": cnt.init_ms, "prepare_s": t_prep, "gq_refine_s": t_dev,
                  "export_s": t_exp,
                  "kernel_launches": int(cnt.kernel_launches), "region_calls": int(cnt.region_calls),
                  "region_ms": cnt.region_ms, "bytes_alg": int(cnt.bytes_alg),
                  "bytes_refine": int(cnt.bytes_refine),
                  "alg_counts": {"n_cand": int(cnt.n_cand), "t_tested": int(cnt.t_tested), "k_claims": int(cnt.k_claims),
                                 "t_created": int(cnt.t_created), "t_deleted": int(cnt.t_deleted)},
                  "exact_calls": [int(x) for x in cnt.exact_calls]}
    if cfg.verbose:
        for r in rep.per_round:
            print("round {round} phase={phase} candidates={candidates} accepted={accepted} blasted={blasted} "
                  "failed={failed} inserted={inserted} workers={workers} time={time:.3f}".format(**r))
    return mesh, rep
