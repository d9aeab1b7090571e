"""Time the host setup of a config (validation, box closure, facet axes) with
the device pair certifier and with the numpy path; check they agree."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03406_b200 import synth
from paper_1903_03406_b200.prepare import prepare, facet_keep
from paper_1903_03406_b200.plc import validate

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
plc = synth.config_plc(name)
for mode in ("device", "host"):
    os.environ["GQM3D_HOST_SETUP"] = "1" if mode == "host" else "0"
    t = time.perf_counter(); v = validate(plc); t1 = time.perf_counter() - t
    t = time.perf_counter(); p = prepare(plc); k = facet_keep(p.plc); t2 = time.perf_counter() - t
    print(f"{name} {mode}: validate {t1:.2f}s ({len(v)} violations) prepare+keep {t2:.2f}s", flush=True)
