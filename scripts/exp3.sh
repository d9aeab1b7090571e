mkdir -p gpurun_out/exp3
timeout 150 python scripts/c3obl.py 2000 20 > gpurun_out/exp3/c3obl.log 2>&1; echo "exit $?" >> gpurun_out/exp3/c3obl.log
GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 150 python scripts/c3obl.py 2000 20 > gpurun_out/exp3/c3obl_dbg.log 2>&1; echo "exit $?" >> gpurun_out/exp3/c3obl_dbg.log
GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 200 python scripts/run_cfg.py C4 --scale 0.02 --level 3 --torus 50,25 --verbose --audit > gpurun_out/exp3/c4_l3.log 2>&1; echo "exit $?" >> gpurun_out/exp3/c4_l3.log
