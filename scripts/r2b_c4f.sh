mkdir -p gpurun_out/r2f
timeout 900 python scripts/run_cfg.py C4 --max-rounds 500 --verbose > gpurun_out/r2f/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2f/c4.log
