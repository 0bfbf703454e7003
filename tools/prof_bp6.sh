#!/bin/bash
# ncu --set full of the three-component DMMA kernels at C4 (BP6 p = 7, 6)
for pd in "7 34" "6 40"; do
  set -- $pd
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmma3_kernel -s 2 -c 1 \
    -o gpurun_out/bp6_p$1 python tools/prof_step.py --bp bp6 --degree $1 --elems $2 --iters 1 > gpurun_out/bp6_prof_p$1.log 2>&1
done
