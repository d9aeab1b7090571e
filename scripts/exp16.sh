mkdir -p gpurun_out/exp16
for L in libgqm3d.so libgqm3d_w4.so libgqm3d_w4m4.so; do
  GQM3D_LIB=paper_1903_03406_b200/$L timeout 120 python scripts/time_lib.py C2 1.0 3 >> gpurun_out/exp16/variants.log 2>&1
  GQM3D_LIB=paper_1903_03406_b200/$L timeout 120 python scripts/time_lib.py C5 1.0 2 >> gpurun_out/exp16/variants.log 2>&1
done
GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_03406_b200 import synth, refine, RefineConfig
plc = synth.triangles_cloud(5000, 40, 0, snapped=False)
mesh, rep = refine(plc, RefineConfig(B=1.4))
print('ok', rep.steiner_points)
" > gpurun_out/exp16/c3obl.log 2>&1; echo "exit $?" >> gpurun_out/exp16/c3obl.log
GQM3D_OBLIQUE_BOX=0 GQ_WATCHDOG=20 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 420 python scripts/run_cfg.py C4 --verbose > gpurun_out/exp16/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp16/c4_nobox.log
