mkdir -p gpurun_out/exp25
GQ_T2_LAUNCHES=1 GQ_PROFILE=3 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp25/c5_launches.log 2>&1
GQ_T2_LAUNCHES=1 GQ_TRACE=1 timeout 300 python scripts/time_lib.py C5 1.0 0 2>&1 | grep "^\[t2\]" > gpurun_out/exp25/c5_t2trace.log
