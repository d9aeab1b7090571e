mkdir -p gpurun_out/r2r
GQM3D_LIB=$PWD/paper_1903_03406_b200/libgqm3d_dbg.so timeout 1200 python scripts/c3obl.py 250000 2000 > gpurun_out/r2r/c3obl_dbg.log 2>&1; echo "exit $?" >> gpurun_out/r2r/c3obl_dbg.log
grep -v "^round\|^  \|noseed" gpurun_out/r2r/c3obl_dbg.log | tail -60 > gpurun_out/r2r/c3obl_dbg_tail.txt
