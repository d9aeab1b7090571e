mkdir -p gpurun_out/r2dd
timeout 300 python scripts/time_lib.py C2 1.0 3 > gpurun_out/r2dd/c2.log 2>&1
timeout 300 python scripts/time_lib.py C5 1.0 2 > gpurun_out/r2dd/c5.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2dd/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2dd/gputests.log
