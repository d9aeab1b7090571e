mkdir -p gpurun_out/r2ee
timeout 1200 python bench.py > gpurun_out/r2ee/bench_c2.log 2>&1; echo "exit $?" >> gpurun_out/r2ee/bench_c2.log
