mkdir -p gpurun_out/exp5
GQ_CAPX=0.01 timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp5/pytest_capx.log 2>&1; echo "exit $?" >> gpurun_out/exp5/pytest_capx.log
GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so GQ_PROFILE=1 timeout 1200 python scripts/run_cfg.py C4 --verbose --audit > gpurun_out/exp5/c4_full.log 2>&1; echo "exit $?" >> gpurun_out/exp5/c4_full.log
