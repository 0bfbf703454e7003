#!/bin/bash
# operator-kernel ablations (measurement only): 1 = no x gather, 2 = no RED scatter, 4 = no qdata stream, 8 = no L2 prefetch of qdata
for a in 0 8 1 2 3; do
  echo -n "ablate=$a "; HXF_ABLATE=$a python bench.py --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('apply_us=%.1f k1_us=%.1f'%(d['apply']['us'], d['cg_iter']['operator_kernel_us']))"
done
