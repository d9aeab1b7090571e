"""Mesh output files, written by the native library.

``write_mesh(mesh, node_path, ele_path, face_path=None)`` has the signature
and produces the same bytes as the reference's
/root/reference/pkg/src/tetrefine/formats.py:245-263 (.node with the origin
attribute, .ele of the alive real tets, .face of the subfaces with their
polygon id; 1-based; coordinates to 17 significant digits), formatted in C++
(gq_write_mesh in libgqm3d.so) instead of one Python f-string per row.
Input parsers (.node/.poly/.smesh) are outside the GPU path.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import IOFailure


def write_mesh(mesh, node_path, ele_path, face_path=None):
    nv, nt = int(mesh.nv), int(mesh.nt)
    pts = np.ascontiguousarray(mesh.points[:nv], dtype=np.float64)
    org = np.ascontiguousarray(mesh.vert_origin[:nv], dtype=np.uint8)
    tv = np.ascontiguousarray(mesh.tv[:nt], dtype=np.int32)
    alive = np.ascontiguousarray(mesh.alive[:nt], dtype=np.uint8)
    faces = None
    nf = 0
    if face_path is not None:
        items = sorted(mesh.subfaces.items())
        faces = np.ascontiguousarray(np.array([(a, b, c, pid) for (a, b, c), pid in items], dtype=np.int32).reshape(-1, 4))
        nf = len(faces)
    st = _native.lib().gq_write_mesh(str(node_path).encode(), str(ele_path).encode(),
                                     None if face_path is None else str(face_path).encode(),
                                     _native._p(pts), _native._p(org), nv, _native._p(tv), _native._p(alive), nt,
                                     None if faces is None else _native._p(faces), nf)
    if st != 0:
        raise IOFailure(f"cannot write {node_path} / {ele_path} / {face_path}")
