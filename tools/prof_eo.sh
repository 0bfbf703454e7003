#!/bin/bash
# ncu --set full of the even-odd tensor-core kernel (BP5 p = 12 and 15)
for pd in "12 18" "15 14"; do
  set -- $pd
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmmaeo -s 2 -c 1 \
    -o gpurun_out/eo_p$1 python tools/prof_step.py --bp bp5 --degree $1 --elems $2 --iters 1 > gpurun_out/eo_prof_p$1.log 2>&1
done
