"""Native .node/.ele/.face writer against a Python restatement of the
reference writer (formats.py:210-263): byte-identical files.  Host code
only, no GPU."""

import numpy as np

from paper_1903_03406_b200.formats import write_mesh
from paper_1903_03406_b200.mesh import Mesh


def _reference_bytes(mesh, tmp):
    F = "{:.17g}".format
    node = [f"{mesh.nv} 3 1 0\n"] + [f"{k + 1} {F(p[0])} {F(p[1])} {F(p[2])} {int(mesh.vert_origin[k])}\n"
                                   for k, p in enumerate(mesh.points[:mesh.nv])]
    tets = mesh.real_tets()
    ele = [f"{len(tets)} 4 0\n"] + [f"{k + 1} " + " ".join(str(int(v) + 1) for v in mesh.tv[t]) + "\n"
                                    for k, t in enumerate(tets)]
    faces = sorted(mesh.subfaces.items())
    face = [f"{len(faces)} 1\n"] + [f"{k + 1} {a + 1} {b + 1} {c + 1} {pid}\n" for k, ((a, b, c), pid) in enumerate(faces)]
    return "".join(node), "".join(ele), "".join(face)


def test_write_mesh_matches_reference_format(tmp_path):
    rng = np.random.default_rng(0)
    nv, nt = 200, 500
    pts = rng.normal(size=(nv, 3)) * np.array([1e-7, 1.0, 3e5])
    pts[3] = (-0.0, 1e-300, np.pi)
    arrays = dict(points=pts, vert_origin=(rng.random(nv) < 0.5).astype(np.uint8), vert_tet=np.zeros(nv, np.int32),
                  tv=rng.integers(0, nv, (nt, 4)).astype(np.int32), tn=np.zeros((nt, 4), np.int32),
                  alive=(rng.random(nt) < 0.7).astype(np.uint8), sub_mask=np.zeros(nt, np.uint8),
                  seg_mask=np.zeros(nt, np.uint8), ratio=np.zeros(nt), skip_flag=np.zeros(nt, np.uint8))
    arrays["tv"][::5, 3] = -1                       # ghosts are not written
    faces = {tuple(sorted(rng.choice(nv, 3, replace=False).tolist())): int(rng.integers(0, 9)) for _ in range(40)}
    mesh = Mesh(arrays, {}, faces, 1.0)
    write_mesh(mesh, tmp_path / "m.node", tmp_path / "m.ele", tmp_path / "m.face")
    want = _reference_bytes(mesh, tmp_path)
    got = tuple((tmp_path / f"m.{e}").read_text() for e in ("node", "ele", "face"))
    assert got == want
    # round trip of the coordinates
    back = np.array([[float(x) for x in line.split()[1:4]] for line in got[0].splitlines()[1:]])
    assert np.array_equal(back, pts)
