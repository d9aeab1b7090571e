mkdir -p gpurun_out/r2s
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2s/gputests.log
GQM3D_LIB=$PWD/paper_1903_03406_b200/libgqm3d_dbg.so timeout 1200 python scripts/c3obl.py 250000 2000 > gpurun_out/r2s/c3obl_dbg.log 2>&1; echo "exit $?" >> gpurun_out/r2s/c3obl_dbg.log
grep -v "^round\|^  \|noseed\|^\[huge\]" gpurun_out/r2s/c3obl_dbg.log | tail -40 > gpurun_out/r2s/c3obl_dbg_tail.txt
grep "^round" gpurun_out/r2s/c3obl_dbg.log | tail -3 >> gpurun_out/r2s/c3obl_dbg_tail.txt
gzip -f gpurun_out/r2s/c3obl_dbg.log
