mkdir -p gpurun_out/r2g
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2g/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2g/gputests.log
timeout 900 python scripts/run_cfg.py C4 --max-rounds 500 --verbose > gpurun_out/r2g/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2g/c4.log
