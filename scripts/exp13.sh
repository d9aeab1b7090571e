mkdir -p gpurun_out/exp13
GQM3D_OBLIQUE_BOX=0 GQ_TRACE=1 GQ_TRACE_FROM=250 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so GQ_PROFILE=1 timeout 700 python scripts/run_cfg.py C4 --verbose --audit > gpurun_out/exp13/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp13/c4_nobox.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp13/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp13/pytest.log
