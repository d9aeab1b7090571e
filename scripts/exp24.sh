mkdir -p gpurun_out/exp24
timeout 120 python scripts/time_lib.py C2 1.0 2 > gpurun_out/exp24/c2.log 2>&1
timeout 600 python scripts/batch_scaling.py 16 > gpurun_out/exp24/scaling.log 2>&1; echo "exit $?" >> gpurun_out/exp24/scaling.log
GQ_PROFILE=3 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp24/c5_stages.log 2>&1
timeout 700 python -m pytest tests -m gpu -x -q > gpurun_out/exp24/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp24/pytest.log
