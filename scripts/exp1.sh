set -x
mkdir -p gpurun_out/exp1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/exp1/smi.txt
timeout 240 python scripts/c3obl.py 2000 20 -v > gpurun_out/exp1/c3obl_2k20.log 2>&1; echo "exit $?" >> gpurun_out/exp1/c3obl_2k20.log
timeout 200 python scripts/run_cfg.py C4 --scale 0.02 --level 3 --torus 50,25 --verbose --audit > gpurun_out/exp1/c4_l3.log 2>&1; echo "exit $?" >> gpurun_out/exp1/c4_l3.log
timeout 200 python scripts/run_cfg.py C3 --scale 0.02 --verbose > gpurun_out/exp1/c3_002.log 2>&1; echo "exit $?" >> gpurun_out/exp1/c3_002.log
