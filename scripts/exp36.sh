mkdir -p gpurun_out/exp36
timeout 1500 python scripts/run_cfg.py C4 --max-rounds 500 --verbose > gpurun_out/exp36/c4.log 2>&1; echo "exit $?" >> gpurun_out/exp36/c4.log
