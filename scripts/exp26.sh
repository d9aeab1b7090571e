mkdir -p gpurun_out/exp26
GQ_PROFILE=1 timeout 120 python scripts/time_lib.py C5 1.0 1 > gpurun_out/exp26/c5.log 2>&1
GQ_PROFILE=1 timeout 120 python scripts/time_lib.py C2 1.0 1 > gpurun_out/exp26/c2.log 2>&1
