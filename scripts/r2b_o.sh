mkdir -p gpurun_out/r2o
timeout 1200 python bench.py > gpurun_out/r2o/bench_c2.log 2>&1; echo "exit $?" >> gpurun_out/r2o/bench_c2.log
timeout 1200 python bench.py --config C5 --north-star-rounds 0 > gpurun_out/r2o/bench_c5.log 2>&1; echo "exit $?" >> gpurun_out/r2o/bench_c5.log
timeout 1200 python bench.py --impl reference > gpurun_out/r2o/bench_ref.log 2>&1; echo "exit $?" >> gpurun_out/r2o/bench_ref.log
