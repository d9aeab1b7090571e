mkdir -p gpurun_out/r2v
timeout 1200 python bench.py > gpurun_out/r2v/bench_c2.log 2>&1; echo "exit $?" >> gpurun_out/r2v/bench_c2.log
