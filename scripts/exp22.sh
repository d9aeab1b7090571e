mkdir -p gpurun_out/exp22
timeout 120 python scripts/time_lib.py C2 1.0 2 > gpurun_out/exp22/c2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp22/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp22/pytest.log
timeout 600 python bench.py --steps 2 --warmup 1 > gpurun_out/exp22/bench_c2.json 2> gpurun_out/exp22/bench_c2.err; echo "exit $?" >> gpurun_out/exp22/bench_c2.err
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/exp22/bench_c5.json 2> gpurun_out/exp22/bench_c5.err; echo "exit $?" >> gpurun_out/exp22/bench_c5.err
