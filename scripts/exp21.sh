mkdir -p gpurun_out/exp21
GQM3D_OBLIQUE_BOX=0 GQ_WATCHDOG=30 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 1300 python scripts/run_cfg.py C4 --verbose --max-rounds 340 > gpurun_out/exp21/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp21/c4_nobox.log
