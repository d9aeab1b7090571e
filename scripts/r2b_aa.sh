mkdir -p gpurun_out/r2aa
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2aa/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2aa/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2aa/smoke.log 2>&1; echo "exit $?" >> gpurun_out/r2aa/smoke.log
timeout 300 python scripts/time_lib.py C5 1.0 1 > gpurun_out/r2aa/c5.log 2>&1
