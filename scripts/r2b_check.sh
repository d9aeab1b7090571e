mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2b/gputests.log
timeout 1800 python scripts/run_cfg.py C4 --max-rounds 500 --verbose > gpurun_out/r2b/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2b/c4.log
