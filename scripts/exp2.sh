mkdir -p gpurun_out/exp2
timeout 150 python scripts/c3obl.py 2000 20 > gpurun_out/exp2/c3obl.log 2>&1; echo "exit $?" >> gpurun_out/exp2/c3obl.log
GQ_TRACE=1 timeout 150 python scripts/run_cfg.py C4 --scale 0.02 --level 3 --torus 50,25 --verbose --audit > gpurun_out/exp2/c4_l3.log 2>&1; echo "exit $?" >> gpurun_out/exp2/c4_l3.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp2/pytest.log
