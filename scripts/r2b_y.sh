mkdir -p gpurun_out/r2y
timeout 600 python scripts/run_cfg.py C4 --max-rounds 200 --verbose > gpurun_out/r2y/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2y/c4.log
