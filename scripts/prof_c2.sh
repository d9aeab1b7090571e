# ncu evidence for the bench kernels (one gpurun call; every ncu run after a plain run exited 0).
# The .ncu-rep files are exported to CSV on the box and dropped (gpurun copies back <= 64 MiB).
mkdir -p gpurun_out/prof
CMD="python scripts/time_lib.py C2 1.0 0"
cap() {   # name kernel-regex skip
  ncu --set full --clock-control none --import-source on -k regex:"^$2" -s $3 -c 1 -f -o gpurun_out/prof/$1 $CMD > gpurun_out/prof/ncu_$1.log 2>&1 || return 1
  ncu -i gpurun_out/prof/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof/$1.ncu-rep --page details --csv > gpurun_out/prof/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/prof/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$1_sass.csv 2>/dev/null
  gzip -f gpurun_out/prof/$1_sass.csv
  rm -f gpurun_out/prof/$1.ncu-rep
}
$CMD > gpurun_out/prof/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/prof/launches_c2.csv $CMD > gpurun_out/prof/ncu_launch.log 2>&1 && \
gzip -f gpurun_out/prof/launches_c2.csv && \
cap region_warp k_region_warp 60 && cap init_stars k_init_stars_warp 200 && cap region_block k_region_block 2 && cap check k_check 20
echo "exit $?" > gpurun_out/prof/exit.txt
du -sh gpurun_out/prof >> gpurun_out/prof/exit.txt
