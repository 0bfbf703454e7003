#!/bin/bash
# Round-2 (second session) ncu captures: the fused PCG step kernel, the
# even-odd kernel (staged / L2 factors), the component-batched BP6 kernel,
# and the bench launch list
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r2b_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pcg_step -s 10 -c 1 -o gpurun_out/r2b_step python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r2b_p1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmmaeo -s 2 -c 1 -o gpurun_out/r2b_eo_p15 python tools/prof_step.py --bp bp5 --degree 15 --elems 14 --iters 1 > gpurun_out/r2b_p2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmmaeo -s 2 -c 1 -o gpurun_out/r2b_eo_p13 python tools/prof_step.py --bp bp5 --degree 13 --elems 17 --iters 1 > gpurun_out/r2b_p3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmma3 -s 2 -c 1 -o gpurun_out/r2b_dmma3_p7 python tools/prof_step.py --bp bp6 --degree 7 --elems 34 --iters 1 > gpurun_out/r2b_p4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmma3 -s 2 -c 1 -o gpurun_out/r2b_dmma3_p6 python tools/prof_step.py --bp bp6 --degree 6 --elems 40 --iters 1 > gpurun_out/r2b_p5.log 2>&1
