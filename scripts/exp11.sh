mkdir -p gpurun_out/exp11
GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so GQ_PROFILE=1 timeout 1200 python scripts/run_cfg.py C4 --verbose --audit > gpurun_out/exp11/c4_full_box.log 2>&1; echo "exit $?" >> gpurun_out/exp11/c4_full_box.log
