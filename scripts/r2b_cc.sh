mkdir -p gpurun_out/r2cc
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_region_warp" -s 4 -c 1 -f -o gpurun_out/r2cc/region_warp python scripts/time_lib.py C2 1.0 1 > gpurun_out/r2cc/ncu.log 2>&1
ncu -i gpurun_out/r2cc/region_warp.ncu-rep --page raw --csv > gpurun_out/r2cc/region_warp_raw.csv 2>/dev/null
ncu -i gpurun_out/r2cc/region_warp.ncu-rep --page details --csv > gpurun_out/r2cc/region_warp_details.csv 2>/dev/null
rm -f gpurun_out/r2cc/region_warp.ncu-rep
