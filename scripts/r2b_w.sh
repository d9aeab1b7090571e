mkdir -p gpurun_out/r2w
for W in 256 1024 128; do
  GQ_FB_WINDOW=$W timeout 600 python scripts/run_cfg.py C4 --max-rounds 500 > gpurun_out/r2w/c4_w$W.log 2>&1
done
