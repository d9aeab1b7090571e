mkdir -p gpurun_out/exp8
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp8/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp8/pytest.log
GQ_CAPX=0.01 timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp8/pytest_capx.log 2>&1; echo "exit $?" >> gpurun_out/exp8/pytest_capx.log
GQM3D_OBLIQUE_BOX=0 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 1500 python scripts/run_cfg.py C4 --verbose --audit > gpurun_out/exp8/c4_full_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp8/c4_full_nobox.log
