"""Step-wise GPU check used during development: predicates, then small
refinements compared with the CPU oracle.  Usage: python scripts/gpu_debug.py [case ...]"""
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
from paper_1903_03406_b200 import _native, synth, RefineConfig, refine  # noqa: E402
from tests.golden.cases import CASES  # noqa: E402

g = np.load(os.path.join(ROOT, "tests/golden/predicates.npz"))
for name, key, inp in (("orient3d", "o3d", "o3d_in"), ("insphere", "isp", "isp_in"), ("orient2d", "o2d", "o2d_in"),
                       ("incircle2d", "icc", "icc_in"), ("incircle3d", "inc3", "inc3_in"),
                       ("encroaches_segment", "eseg", "eseg_in"), ("encroaches_face", "eface", "eface_in")):
    try:
        out = _native.batch(name, g[inp])
        print(f"pred {name}: {'OK' if np.array_equal(out, g['out_' + key]) else 'MISMATCH %d' % int((out != g['out_' + key]).sum())}", flush=True)
    except Exception as e:
        print("pred", name, "ERROR", e, flush=True)

cases = sys.argv[1:] or ["cube0", "cube100"]
for name in cases:
    build, B = CASES[name]
    plc = build()
    try:
        t = time.time()
        mesh, rep = refine(plc, RefineConfig(B=B))
        dt = time.time() - t
        ref = oracle.refine(plc, B=B)
        st_o = int((ref["vert_origin"] == 1).sum())
        same = mesh.nv == ref["nv"] and np.array_equal(mesh.points, ref["points"])
        print(f"{name}: gpu steiner {rep.steiner_points} bad {rep.bad_tet_count} rounds {len(rep.per_round)} "
              f"| oracle steiner {st_o} rounds {len(ref['per_round'])} | identical points {same} | "
              f"wall {dt:.2f}s device {rep.device['device_ms']:.1f}ms init {rep.device['init_ms']:.1f}ms "
              f"launches {rep.device['kernel_launches']}", flush=True)
        for a, b in zip(rep.per_round, ref["per_round"]):
            ka = {k: a[k] for k in ("phase", "candidates", "accepted", "blasted", "failed", "inserted", "pending_segments", "pending_faces")}
            kb = {k: b[k] for k in ka}
            if ka != kb:
                print("  first round diff", a["round"], "\n   gpu   ", ka, "\n   oracle", kb, flush=True)
                break
        try:
            mesh.audit()
            print("  audit ok", flush=True)
        except AssertionError as e:
            print("  AUDIT FAIL", e, flush=True)
    except Exception as e:
        print(name, "ERROR", e, flush=True)
        traceback.print_exc()
