mkdir -p gpurun_out/r2l
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2l/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2l/gputests.log
timeout 900 python scripts/run_cfg.py C4 --max-rounds 500 --verbose > gpurun_out/r2l/c4.log 2>&1; echo "exit $?" >> gpurun_out/r2l/c4.log
GQ_PROFILE=3 timeout 300 python scripts/time_lib.py C1 1.0 3 > gpurun_out/r2l/c1_prof.log 2>&1
GQ_PROFILE=2 timeout 300 python scripts/time_lib.py C1 1.0 3 > gpurun_out/r2l/c1_prof2.log 2>&1
timeout 300 python scripts/time_lib.py C1 1.0 3 > gpurun_out/r2l/c1.log 2>&1
