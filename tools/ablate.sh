#!/bin/bash
# operator-kernel ablations (measurement only; timed single applies):
# 1 = no x gather (per-lane path), 2 = no RED scatter, 4 = no qdata stream,
# 16 = no contraction / QFunction arithmetic (DMMA kernel)
for a in ${ABL:-0 16 4 20 2 18}; do
  HXF_ABLATE=$a python tools/k1_time.py ${K1ARGS:-} --tag "ablate=$a"
done
