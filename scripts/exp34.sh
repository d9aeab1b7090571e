mkdir -p gpurun_out/exp34
for cfg in "C1 1.0" "C5 1.0" "C2 1.0"; do
  timeout 120 python scripts/time_lib.py $cfg 2 > gpurun_out/exp34/new_${cfg% *}.log 2>&1
  GQ_GRID_THREAD=1 GQ_T2_THREAD=1 timeout 120 python scripts/time_lib.py $cfg 2 > gpurun_out/exp34/old_${cfg% *}.log 2>&1
done
GQ_PROFILE=3 timeout 120 python scripts/time_lib.py C1 1.0 1 > gpurun_out/exp34/c1p3.log 2>&1
