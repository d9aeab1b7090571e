mkdir -p gpurun_out/exp27
GQ_PROFILE=3 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp27/c5.log 2>&1
GQ_PROFILE=3 GQ_T2_LAUNCHES=1 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp27/c5l.log 2>&1
