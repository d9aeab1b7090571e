mkdir -p gpurun_out/exp33
GQ_PROFILE=3 timeout 120 python scripts/time_lib.py C1 1.0 1 > gpurun_out/exp33/c1p3.log 2>&1
GQ_PROFILE=2 timeout 120 python scripts/time_lib.py C1 1.0 1 > gpurun_out/exp33/c1p2.log 2>&1
timeout 300 nsys --version > /dev/null 2>&1 || true
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp33/c1_launches.csv python scripts/time_lib.py C1 1.0 0 > gpurun_out/exp33/ncu.log 2>&1
gzip -f gpurun_out/exp33/c1_launches.csv
