#!/bin/bash
# C2 timing bundle for a gpurun call: plain runs, coarse profile, init trace
mkdir -p gpurun_out
for i in 1 2 3; do python scripts/run_c2.py ${SCALE:-1.0} 2>&1 | grep "^C2"; done
GQ_PROFILE=1 python scripts/run_c2.py ${SCALE:-1.0} 2>&1 | grep "gq profile"
GQ_PROFILE=3 python scripts/run_c2.py ${SCALE:-1.0} 2>&1 | grep "gq fine"
GQ_TRACE=1 python scripts/run_c2.py ${SCALE:-1.0} > gpurun_out/trace.log 2>&1
grep "^\[init\]" gpurun_out/trace.log | awk '{w+=$5; b+=$7; if ($7>0) nb++} END {print "init rounds", NR, "sumW", w, "big", b, "rounds with big", nb}'
