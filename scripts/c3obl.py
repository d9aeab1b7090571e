import sys, time; sys.path.insert(0, ".")
from paper_1903_03406_b200 import synth, refine, RefineConfig
n = int(sys.argv[1]) if len(sys.argv) > 1 else 250000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
plc = synth.triangles_cloud(n, m, 0, snapped=False)
t = time.time()
mesh, rep = refine(plc, RefineConfig(B=1.4, verbose=True))
print("C3-oblique", n, m, "steiner", rep.steiner_points, "bad", rep.bad_tet_count, "rounds", len(rep.per_round),
      "dev ms", rep.device["device_ms"], "wall", time.time() - t, flush=True)
if "--audit" in sys.argv:
    mesh.audit(); print("audit ok")
