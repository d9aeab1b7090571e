mkdir -p gpurun_out/exp20
timeout 120 python scripts/time_lib.py C2 1.0 2 > gpurun_out/exp20/c2.log 2>&1
timeout 300 python scripts/c3obl.py 5000 40 > gpurun_out/exp20/c3obl.log 2>&1; echo "exit $?" >> gpurun_out/exp20/c3obl.log
GQM3D_OBLIQUE_BOX=0 GQ_WATCHDOG=30 timeout 1000 python scripts/run_cfg.py C4 --verbose > gpurun_out/exp20/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp20/c4_nobox.log
