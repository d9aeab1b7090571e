mkdir -p gpurun_out/r2z
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2z/gputests.log 2>&1; echo "exit $?" >> gpurun_out/r2z/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z/smoke.log 2>&1; echo "exit $?" >> gpurun_out/r2z/smoke.log
