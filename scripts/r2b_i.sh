mkdir -p gpurun_out/r2i
timeout 300 python scripts/run_cfg.py C4 --max-rounds 200 --verbose > gpurun_out/r2i/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2i/c4.log
timeout 1200 python bench.py > gpurun_out/r2i/bench.log 2>&1; echo "exit $?" >> gpurun_out/r2i/bench.log
