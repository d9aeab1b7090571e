mkdir -p gpurun_out/exp29
GQ_PROFILE=3 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp29/c5w.log 2>&1
GQ_PROFILE=3 GQ_T2_THREAD=1 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp29/c5t.log 2>&1
GQ_PROFILE=3 GQ_T2_FUSED_MAX=0 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp29/c5w0.log 2>&1
timeout 120 python scripts/time_lib.py C2 1.0 2 > gpurun_out/exp29/c2.log 2>&1
timeout 120 python scripts/time_lib.py C3 0.2 1 > gpurun_out/exp29/c3.log 2>&1
