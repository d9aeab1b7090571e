mkdir -p gpurun_out/exp30
timeout 900 python bench.py > gpurun_out/exp30/bench_c2.json 2> gpurun_out/exp30/bench_c2.err; echo "exit $?" >> gpurun_out/exp30/bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/exp30/bench_ref.json 2> gpurun_out/exp30/bench_ref.err; echo "exit $?" >> gpurun_out/exp30/bench_ref.err
timeout 900 python bench.py --config C5 > gpurun_out/exp30/bench_c5.json 2> gpurun_out/exp30/bench_c5.err; echo "exit $?" >> gpurun_out/exp30/bench_c5.err
timeout 1500 bash scripts/prof_c2.sh
