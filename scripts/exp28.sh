mkdir -p gpurun_out/exp28
GQ_T2_LAUNCHES=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_t2 --csv --log-file gpurun_out/exp28/t2.csv python scripts/time_lib.py C5 1.0 0 > gpurun_out/exp28/run.log 2>&1
GQ_T2_LAUNCHES=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_t2_compute --launch-skip 520 -c 1 -o gpurun_out/exp28/t2c python scripts/time_lib.py C5 1.0 0 > gpurun_out/exp28/run2.log 2>&1
GQ_T2_LAUNCHES=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_t2_commit --launch-skip 520 -c 1 -o gpurun_out/exp28/t2m python scripts/time_lib.py C5 1.0 0 > gpurun_out/exp28/run3.log 2>&1
