import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03406_b200 import synth, refine, RefineConfig
n = int(sys.argv[1])
mesh, rep = refine(synth.cube_points(n, 0), RefineConfig(B=2.0, max_rounds=int(sys.argv[2]) if len(sys.argv) > 2 else 500))
print("ok steiner", rep.steiner_points, "rounds", len(rep.per_round), flush=True)
