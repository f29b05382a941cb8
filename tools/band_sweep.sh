#!/bin/bash
# Strip width sweep of the band processing order (HX_BAND_STRIP, columns) on one workload: cold build time.
WL=${1:-C4}
for w in ${STRIPS:-0 4096 8192 16384 32768 65536}; do
  echo -n "strip=$w  "; HX_BAND_STRIP=$w python tools/asm_time.py --one $WL
done
