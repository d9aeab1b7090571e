mkdir -p gpurun_out/exp15
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp15/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp15/pytest.log
GQM3D_OBLIQUE_BOX=0 GQ_WATCHDOG=20 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 600 python scripts/run_cfg.py C4 --verbose > gpurun_out/exp15/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp15/c4_nobox.log
