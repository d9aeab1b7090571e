"""The sequential fallback (refine.py:748-806, called in failed-list order at
refine.py:897-902) runs on the device in waves: a side-effect-free parallel
evaluation of every remaining failed candidate, then an in-order application
up to the first candidate that inserts, a window of candidates per wave
(gq_fallback.cuh).  These tests run the
same refinements with the one-thread loop (GQ_FALLBACK_SERIAL=1, read when the
library loads, hence a subprocess per mode) and require identical meshes:
points, tets, constraint sets, per-round rows and the skip list."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WORKER = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1903_03406_b200 import synth, refine, RefineConfig
case = sys.argv[2]
if case == "oblique":
    plc, B = synth.triangles_cloud(5000, 40, 0, snapped=False), 1.4
elif case == "c2":
    plc, B = synth.config_plc("C2", scale=0.1), 1.6
else:   # C4's shape (nested icospheres + torus + interior points), small
    plc, B = synth.nested_surfaces(20000, level=3, torus=(40, 20)), 1.5
mesh, rep = refine(plc, RefineConfig(B=B, max_rounds=200))
h = hashlib.sha256()
for a in (mesh.points, mesh.tv, mesh.tn, mesh.alive):
    h.update(np.ascontiguousarray(a).tobytes())
rows = [[int(r[k]) for k in ("round", "candidates", "accepted", "blasted", "failed", "inserted")] for r in rep.per_round]
print(json.dumps({"hash": h.hexdigest(), "steiner": rep.steiner_points, "rows": rows,
                  "subfaces": sorted(map(list, mesh.subfaces)), "subsegments": sorted(map(list, mesh.subsegments)),
                  "skipped": [[s["kind"], s["reason"], list(s["vertices"])] for s in rep.skipped]}))
"""


def _run(case: str, serial: bool, window: int = 0) -> dict:
    env = dict(os.environ)
    env.pop("GQ_FALLBACK_SERIAL", None)
    env.pop("GQ_FB_WINDOW", None)
    if serial:
        env["GQ_FALLBACK_SERIAL"] = "1"
    if window:
        env["GQ_FB_WINDOW"] = str(window)
    out = subprocess.run([sys.executable, "-c", _WORKER, ROOT, case], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("case", ["oblique", "c2", "nested"])
def test_fallback_waves_equal_serial_loop(case):
    waves = _run(case, serial=False)
    serial = _run(case, serial=True)
    narrow = _run(case, serial=False, window=3)    # many windows without a break
    assert narrow["hash"] == serial["hash"] and narrow["rows"] == serial["rows"]
    assert narrow["skipped"] == serial["skipped"]
    if case != "c2":
        assert sum(r[4] for r in waves["rows"]) > 0, "no failed candidate: the fallback was not exercised"
    assert waves["rows"] == serial["rows"]
    assert waves["steiner"] == serial["steiner"]
    assert waves["hash"] == serial["hash"]
    assert waves["subfaces"] == serial["subfaces"]
    assert waves["subsegments"] == serial["subsegments"]
    assert waves["skipped"] == serial["skipped"]
