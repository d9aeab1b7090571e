#!/bin/bash
# compare library variants on C2: device time and region stages (event profile)
for lib in "$@"; do
  echo "== $lib"
  GQM3D_LIB=$PWD/paper_1903_03406_b200/$lib GQ_PROFILE=3 timeout 200 python scripts/run_c2.py 1.0 2 2>&1 | grep "gq fine\|^C2" | tail -2 | sed 's/.*device_ms.: \([0-9.]*\).*/dev \1/; s/.*\(i.region [0-9.]*\).*\(g.warp [0-9.]*\).*\(g.block [0-9.]*\).*/\1 \2 \3/'
done
