mkdir -p gpurun_out/r2t
for L in libgqm3d.so libgqm3d_minb2.so libgqm3d_w4.so libgqm3d.so; do
  echo "== $L" >> gpurun_out/r2t/variants.log
  GQM3D_LIB=$PWD/paper_1903_03406_b200/$L timeout 300 python scripts/time_lib.py C2 1.0 3 >> gpurun_out/r2t/variants.log 2>&1
done
