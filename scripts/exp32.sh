mkdir -p gpurun_out/exp32
timeout 120 python scripts/time_lib.py C2 1.0 2 > gpurun_out/exp32/c2.log 2>&1
timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp32/c5.log 2>&1
timeout 120 python scripts/time_lib.py C1 1.0 2 > gpurun_out/exp32/c1.log 2>&1
timeout 700 python -m pytest tests -m gpu -x -q > gpurun_out/exp32/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp32/pytest.log
