mkdir -p gpurun_out/r2p
timeout 2400 python scripts/run_cfg.py C4 --max-rounds 4000 --verbose > gpurun_out/r2p/c4_long.log 2>&1; echo "exit $?" >> gpurun_out/r2p/c4_long.log
grep -v "^  " gpurun_out/r2p/c4_long.log | grep -v "^\[" | gzip > gpurun_out/r2p/c4_long_rounds.log.gz
