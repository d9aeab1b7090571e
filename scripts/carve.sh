#!/bin/bash
for cv in ${CVS:-0 -1 50 75 100}; do
  echo -n "carveout $cv: "
  GQ_CARVEOUT=$cv GQ_PROFILE=3 timeout 100 python scripts/run_c2.py 1.0 2 2>&1 | grep "gq fine\|^C2" | tail -2 | tr '\n' ' ' | sed 's/.*\(i.region [0-9.]*\).*\(g.warp [0-9.]*\).*device_ms.: \([0-9.]*\).*/\1 \2 dev \3/'
  echo
done
