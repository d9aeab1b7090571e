# ncu evidence for the bench kernels (one gpurun call; every ncu run after a plain run exited 0)
mkdir -p gpurun_out/prof
CMD="python scripts/time_lib.py C2 1.0 0"
$CMD > gpurun_out/prof/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/prof/launches_c2.csv $CMD > gpurun_out/prof/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_region_warp" -s 60 -c 1 -f -o gpurun_out/prof/region_warp $CMD > gpurun_out/prof/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_init_stars_warp" -s 200 -c 1 -f -o gpurun_out/prof/init_stars $CMD > gpurun_out/prof/ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_region_block" -s 2 -c 1 -f -o gpurun_out/prof/region_block $CMD > gpurun_out/prof/ncu3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_check" -s 20 -c 1 -f -o gpurun_out/prof/check $CMD > gpurun_out/prof/ncu4.log 2>&1
echo "exit $?" > gpurun_out/prof/exit.txt
