mkdir -p gpurun_out/exp19
for L in libgqm3d_r1.so libgqm3d.so; do GQM3D_LIB=paper_1903_03406_b200/$L timeout 120 python scripts/time_lib.py C2 1.0 3 >> gpurun_out/exp19/c2.log 2>&1; done
GQ_TRACE=1 GQ_TRACE_FROM=100000 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 200 python scripts/c3obl.py 5000 40 > gpurun_out/exp19/c3obl.log 2>&1; echo "exit $?" >> gpurun_out/exp19/c3obl.log
GQM3D_OBLIQUE_BOX=0 GQM3D_LIB=paper_1903_03406_b200/libgqm3d_dbg.so timeout 300 python scripts/run_cfg.py C4 --verbose --max-rounds 40 > gpurun_out/exp19/c4_nobox.log 2>&1; echo "exit $?" >> gpurun_out/exp19/c4_nobox.log
