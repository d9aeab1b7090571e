mkdir -p gpurun_out/r2m
timeout 900 python -m pytest tests/test_gpu_fallback_waves.py -x -q > gpurun_out/r2m/waves.log 2>&1; echo "exit $?" >> gpurun_out/r2m/waves.log
timeout 900 python scripts/run_cfg.py C4 --max-rounds 500 --verbose > gpurun_out/r2m/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2m/c4.log
