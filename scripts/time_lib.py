"""Device time of a config's refine with the library in GQM3D_LIB (experiments)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03406_b200 import synth, _native
from paper_1903_03406_b200.prepare import prepare, facet_keep
name = sys.argv[1]; scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
B = {"C1": 2.0, "C2": 1.6, "C3": 1.4, "C4": 1.5, "C5": 1.5}[name]
plc = synth.config_plc(name, scale=scale) if name != "C5" else synth.cube_points(int(50000 * scale), 0)
prep = prepare(plc); keep = facet_keep(prep.plc)
ctx = _native.Context(0)
for r in range(reps + 1):
    c = ctx.refine(prep, keep, B, 500, 0)
    if r:
        print(f"{os.path.basename(_native.lib_path())} {name} x{scale}: steiner {c.steiner_points} rounds {c.n_rounds} "
              f"device {c.device_ms:.1f} ms region {c.region_ms:.1f} ms init {c.init_ms:.1f} ms launches {c.kernel_launches}", flush=True)
