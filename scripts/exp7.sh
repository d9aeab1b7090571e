mkdir -p gpurun_out/exp7
GQM3D_OBLIQUE_BOX=0 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 1500 python scripts/run_cfg.py C4 --verbose --audit > gpurun_out/exp7/c4_full_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp7/c4_full_nobox.log
GQ_CAPX=0.01 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 400 python -m pytest tests -m gpu -x -q -k c2_full > gpurun_out/exp7/pytest_capx.log 2>&1; echo "exit $?" >> gpurun_out/exp7/pytest_capx.log
