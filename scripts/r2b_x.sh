mkdir -p gpurun_out/r2x
timeout 900 python -m pytest tests/test_gpu_fallback_waves.py -x -q > gpurun_out/r2x/waves.log 2>&1; echo "exit $?" >> gpurun_out/r2x/waves.log
timeout 600 python scripts/run_cfg.py C4 --max-rounds 500 > gpurun_out/r2x/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2x/c4.log
