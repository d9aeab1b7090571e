"""Run one BASELINE config (optionally scaled / with a custom generator) through refine()."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1903_03406_b200 import synth, refine, RefineConfig
from paper_1903_03406_b200.prepare import prepare

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--level", type=int, default=6)
ap.add_argument("--torus", default="200,100")
ap.add_argument("--B", type=float, default=None)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--audit", action="store_true")
ap.add_argument("--max-rounds", type=int, default=500)
ap.add_argument("--verbose", action="store_true")
ap.add_argument("--filter", default="greedy")
a = ap.parse_args()
Bdef = {"C1": 2.0, "C2": 1.6, "C3": 1.4, "C4": 1.5, "C5": 1.5}[a.config]
B = a.B or Bdef
t = time.time()
if a.config == "C4":
    plc = synth.nested_surfaces(int(1000000 * a.scale), level=a.level, torus=tuple(int(x) for x in a.torus.split(",")))
else:
    plc = synth.config_plc(a.config, scale=a.scale)
print(f"{a.config}: {len(plc.points)} points {len(plc.segments)} segments {len(plc.polygons)} polygons, gen {time.time()-t:.1f}s", flush=True)
for r in range(a.reps):
    t = time.time()
    mesh, rep = refine(plc, RefineConfig(B=B, max_rounds=a.max_rounds, verbose=a.verbose, filter=a.filter))
    dt = time.time() - t
    ph = {}
    for row in rep.per_round:
        ph[row["phase"]] = ph.get(row["phase"], 0) + 1
    print(f"steiner {rep.steiner_points} bad {rep.bad_tet_count} tets {rep.tet_count} rounds {len(rep.per_round)} {ph} "
          f"skipped {len(rep.skipped)} wall {dt:.2f}s dev {rep.device['device_ms']:.0f}ms init {rep.device['init_ms']:.0f}ms "
          f"prepare {rep.device['prepare_s']:.1f}s launches {rep.device['kernel_launches']} "
          f"steiner/s dev {rep.steiner_points / (rep.device['device_ms'] / 1000):.0f} e2e {rep.steiner_points / dt:.0f}", flush=True)
if a.audit:
    t = time.time()
    mesh.audit()
    print(f"audit ok {time.time()-t:.1f}s", flush=True)
