mkdir -p gpurun_out/exp35
CMD="python scripts/time_lib.py C1 1.0 0"
ncu --set full --clock-control none --import-source on -k regex:"^k_t2_fused" -s 60 -c 1 -f -o gpurun_out/exp35/t2f $CMD > gpurun_out/exp35/ncu.log 2>&1
ncu -i gpurun_out/exp35/t2f.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/exp35/t2f_cs.csv 2>/dev/null
ncu -i gpurun_out/exp35/t2f.ncu-rep --page raw --csv > gpurun_out/exp35/t2f_raw.csv 2>/dev/null
gzip -f gpurun_out/exp35/t2f_cs.csv; rm -f gpurun_out/exp35/t2f.ncu-rep
GQ_TRACE=1 timeout 300 python scripts/time_lib.py C1 1.0 0 2>&1 | grep "^\[t2\]" > gpurun_out/exp35/c1_t2trace.log
