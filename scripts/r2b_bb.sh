mkdir -p gpurun_out/r2bb
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2bb/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2bb/gputests.log
timeout 300 python scripts/time_lib.py C2 1.0 3 > gpurun_out/r2bb/c2.log 2>&1
timeout 300 python scripts/time_lib.py C1 1.0 3 > gpurun_out/r2bb/c1.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bb/smoke.log 2>&1; echo "exit $?" >> gpurun_out/r2bb/smoke.log
