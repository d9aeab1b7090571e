mkdir -p gpurun_out/exp17
timeout 120 python scripts/time_lib.py C2 1.0 3 > gpurun_out/exp17/c2.log 2>&1
timeout 200 python scripts/c3obl.py 5000 40 > gpurun_out/exp17/c3obl.log 2>&1; echo "exit $?" >> gpurun_out/exp17/c3obl.log
GQM3D_OBLIQUE_BOX=0 GQ_WATCHDOG=20 timeout 900 python scripts/run_cfg.py C4 --verbose --audit > gpurun_out/exp17/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp17/c4_nobox.log
