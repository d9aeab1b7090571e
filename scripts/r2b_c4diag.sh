mkdir -p gpurun_out/r2c
timeout 900 python scripts/run_cfg.py C4 --max-rounds 190 --verbose > gpurun_out/r2c/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2c/c4.log
