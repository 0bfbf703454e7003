#!/bin/bash
# A/B: component-batched three-component DMMA kernel (op_dmma3.cuh) vs op_dmma.cuh, C4 p = 6, 7
for r in 1 2; do for M in 1 0; do for pd in "7 34" "6 40"; do set -- $pd
  HXF_DMMA3=$M python tools/k1_time.py --bp bp6 --degree $1 --elems $2 --reps 10 --tag "DMMA3=$M"
done; done; done
