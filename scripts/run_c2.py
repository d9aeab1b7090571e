import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03406_b200 import synth, refine, RefineConfig
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
plc = synth.config_plc("C2", scale=scale)
for _ in range(reps):
    t = time.time()
    mesh, rep = refine(plc, RefineConfig(B=1.6, verbose=False))
    dt = time.time() - t
    print(f"C2 x{scale}: steiner {rep.steiner_points} bad {rep.bad_tet_count} tets {rep.tet_count} rounds {len(rep.per_round)} "
          f"skipped {len(rep.skipped)} wall {dt:.2f}s dev {rep.device}", flush=True)
tt = {}
for r in rep.per_round:
    tt[r["phase"]] = tt.get(r["phase"], 0) + r["time"]
print("phase time", tt)
for r in rep.per_round[::10]:
    print(r)
