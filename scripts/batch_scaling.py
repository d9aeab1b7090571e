"""C5-style batch on one GPU: wall time of refine_batch for 1/2/4/8 PLCs in flight."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03406_b200 import synth, RefineConfig
from paper_1903_03406_b200.prepare import prepare, facet_keep
from paper_1903_03406_b200.replicas import refine_batch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
plcs = [synth.cube_points(50000, s) for s in range(n)]
preps = [prepare(p) for p in plcs]; keeps = [facet_keep(p.plc) for p in preps]
cfg = RefineConfig(B=1.5)
refine_batch(plcs[:8], cfg, 0, 8, prepared=(preps[:8], keeps[:8]))   # warm every context
for k in (1, 2, 4, 8, 16):
    t = time.perf_counter()
    cnts = refine_batch(plcs, cfg, 0, k, prepared=(preps, keeps))
    dt = time.perf_counter() - t
    st = sum(int(c.steiner_points) for c in cnts)
    print(f"streams {k}: {n} PLCs in {dt:.2f} s, {st / dt:.0f} Steiner/s, mean device {sum(c.device_ms for c in cnts) / n:.0f} ms", flush=True)
