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
for spec in cases:
    name, _, mr = spec.partition(":")
    max_rounds = int(mr) if mr else 500
    build, B = CASES[name]
    plc = build()
    try:
        t = time.time()
        mesh, rep = refine(plc, RefineConfig(B=B, max_rounds=max_rounds))
        dt = time.time() - t
        ref = oracle.refine(plc, B=B, max_rounds=max_rounds)
        ga = {tuple(r) for r in mesh.tv[mesh.alive == 1].tolist()}
        oa = {tuple(r) for r in ref["tv"][ref["alive"] == 1].tolist()}
        gs = {tuple(sorted(r)) for r in ga}
        os_ = {tuple(sorted(r)) for r in oa}
        print(f"  tets: gpu {len(ga)} oracle {len(oa)}; ordered-equal {ga == oa}; as-sets-equal {gs == os_}; "
              f"ordered diff {len(ga - oa)}; set diff {len(gs - os_)}", flush=True)
        gsub = set(map(tuple, np.asarray(sorted(mesh.subfaces.items())).reshape(-1, 2).tolist())) if False else {k + (v,) for k, v in mesh.subfaces.items()}
        osub = {tuple(r) for r in ref["subfaces"].tolist()}
        print(f"  subfaces gpu {len(gsub)} oracle {len(osub)} only-gpu {sorted(gsub - osub)[:6]} only-oracle {sorted(osub - gsub)[:6]}", flush=True)
        gseg = {k + (v,) for k, v in mesh.subsegments.items()}
        oseg = {tuple(r) for r in ref["subsegments"].tolist()}
        print(f"  subsegs gpu {len(gseg)} oracle {len(oseg)} only-gpu {sorted(gseg - oseg)[:6]} only-oracle {sorted(oseg - gseg)[:6]}", flush=True)
        if gs != os_:
            print("   tets only-gpu", sorted(gs - os_)[:6], "only-oracle", sorted(os_ - gs)[:6], flush=True)
        if gs == os_ and ga != oa:
            ex = sorted(ga - oa)[:3]
            for e in ex:
                k = tuple(sorted(e))
                o = [x for x in oa if tuple(sorted(x)) == k]
                print("   gpu", e, "oracle", o, flush=True)
        st_o = int((ref["vert_origin"] == 1).sum())
        same = mesh.nv == ref["nv"] and np.array_equal(mesh.points, ref["points"])
        print(f"{name}: gpu steiner {rep.steiner_points} bad {rep.bad_tet_count} rounds {len(rep.per_round)} "
              f"| oracle steiner {st_o} rounds {len(ref['per_round'])} | identical points {same} | "
              f"wall {dt:.2f}s device {rep.device['device_ms']:.1f}ms init {rep.device['init_ms']:.1f}ms "
              f"launches {rep.device['kernel_launches']}", flush=True)
        if not same and mesh.nv == ref["nv"]:
            d = np.flatnonzero(np.any(mesh.points != ref["points"], axis=1))
            A = {tuple(r) for r in mesh.points.tolist()}; Bs = {tuple(r) for r in ref["points"].tolist()}
            print(f"  {len(d)} rows differ, first {d[:5].tolist()}; same set {A == Bs}; |A-B|={len(A - Bs)}", flush=True)
            if len(d):
                i = d[0]
                print("   gpu", mesh.points[i].tolist(), "oracle", ref["points"][i].tolist(), flush=True)
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
