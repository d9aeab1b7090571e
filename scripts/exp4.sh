mkdir -p gpurun_out/exp4
export GQ_CAPX=4
GQM3D_OBLIQUE_BOX=0 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 300 python scripts/run_cfg.py C4 --scale 0.02 --level 3 --torus 50,25 --verbose --audit > gpurun_out/exp4/c4_l3_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp4/c4_l3_nobox.log
GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 300 python scripts/run_cfg.py C4 --scale 0.02 --level 3 --torus 50,25 --verbose --audit > gpurun_out/exp4/c4_l3_box.log 2>&1; echo "exit $?" >> gpurun_out/exp4/c4_l3_box.log
timeout 200 python scripts/c3obl.py 25000 200 > gpurun_out/exp4/c3obl_25k.log 2>&1; echo "exit $?" >> gpurun_out/exp4/c3obl_25k.log
