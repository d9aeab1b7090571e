mkdir -p gpurun_out/r2k
timeout 900 python -m pytest tests/test_gpu_fallback_waves.py -x -q > gpurun_out/r2k/waves.log 2>&1; echo "exit $?" >> gpurun_out/r2k/waves.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/r2k/launches_c2.csv python scripts/time_lib.py C2 1.0 1 > gpurun_out/r2k/ncu.log 2>&1; echo "exit $?" >> gpurun_out/r2k/ncu.log
gzip -f gpurun_out/r2k/launches_c2.csv
