mkdir -p gpurun_out/r2e
GQM3D_OBLIQUE_BOX=0 timeout 900 python scripts/run_cfg.py C4 --max-rounds 500 --verbose --audit > gpurun_out/r2e/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/r2e/c4_nobox.log
