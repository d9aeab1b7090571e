mkdir -p gpurun_out/exp6
GQ_CAPX=0.01 timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/exp6/pytest_capx.log 2>&1; echo "exit $?" >> gpurun_out/exp6/pytest_capx.log
GQM3D_OBLIQUE_BOX=0 GQ_PROFILE=1 timeout 1500 python scripts/run_cfg.py C4 --verbose --audit > gpurun_out/exp6/c4_full_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp6/c4_full_nobox.log
