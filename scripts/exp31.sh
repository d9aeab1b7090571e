mkdir -p gpurun_out/exp31
CMD="python scripts/time_lib.py C2 1.0 0"
GQ_PROFILE=3 timeout 120 python scripts/time_lib.py C2 1.0 1 > gpurun_out/exp31/c2prof.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_region_warp" -s 60 -c 1 -f -o gpurun_out/exp31/rw $CMD > gpurun_out/exp31/ncu.log 2>&1
ncu -i gpurun_out/exp31/rw.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/exp31/rw_cs.csv 2>/dev/null
gzip -f gpurun_out/exp31/rw_cs.csv; rm -f gpurun_out/exp31/rw.ncu-rep
