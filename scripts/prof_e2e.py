import sys, os, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03406_b200 import synth, refine, RefineConfig
plc = synth.config_plc("C2")
refine(plc, RefineConfig(B=1.6))
pr = cProfile.Profile(); pr.enable()
t = time.time(); mesh, rep = refine(plc, RefineConfig(B=1.6)); dt = time.time() - t
pr.disable()
print("wall", dt, rep.device)
pstats.Stats(pr).sort_stats('tottime').print_stats(15)
