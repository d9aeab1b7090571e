#!/bin/bash
for wf in ${WFS:-0.125 0.0625 0.03125}; do
  for i in 1 2; do
    echo -n "wf $wf: "; GQ_INIT_WINDOW=$wf python scripts/run_c2.py 1.0 2>&1 | grep "^C2" | sed 's/.*tets \([0-9]*\).*device_ms.: \([0-9.]*\), .init_ms.: \([0-9.]*\).*region_calls.: \([0-9]*\).*/tets \1 dev \2 init \3 regions \4/'
  done
  GQ_INIT_WINDOW=$wf GQ_TRACE=1 python scripts/run_c2.py 1.0 2>&1 | grep "^\[init\]" | awk '{w+=$5; b+=$7; if ($7>0) nb++} END {print "   init rounds", NR, "sumW", w, "big", b, "rounds with big", nb}'
done
