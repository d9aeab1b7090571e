mkdir -p gpurun_out/r2q
timeout 1200 python scripts/c3obl.py 250000 2000 > gpurun_out/r2q/c3obl_full.log 2>&1; echo "exit $?" >> gpurun_out/r2q/c3obl_full.log
timeout 600 python scripts/run_cfg.py C3 --audit > gpurun_out/r2q/c3_snapped_full.log 2>&1; echo "exit $?" >> gpurun_out/r2q/c3_snapped_full.log
