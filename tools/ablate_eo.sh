#!/bin/bash
# Ablations of the even-odd tensor-core kernel (HXF_ABLATE bits: 1 gather,
# 2 scatter, 4 factors, 16 tensor-core products); single applies at ~1e7 DOFs
for cfg in "bp5 15 14" "bp5 13 17" "bp6 13 12"; do
  set -- $cfg
  for A in 0 1 2 4 16 7 23; do
    HXF_ABLATE=$A python tools/k1_time.py --bp $1 --degree $2 --elems $3 --reps 20 --tag "ablate=$A"
  done
done
