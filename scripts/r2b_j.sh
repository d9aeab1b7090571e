mkdir -p gpurun_out/r2j
GQM3D_LIB=$PWD/paper_1903_03406_b200/libgqm3d_dbg.so timeout 600 python scripts/run_cfg.py C4 --max-rounds 170 --verbose > gpurun_out/r2j/c4dbg.log 2>&1; echo "exit $?" >> gpurun_out/r2j/c4dbg.log
