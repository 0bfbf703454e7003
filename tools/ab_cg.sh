#!/bin/bash
# A/B CG-loop options: serpentine sweeps x per-iteration timing events
for cfg in "1 1" "0 1" "1 0" "0 0"; do
  set -- $cfg
  echo -n "serpentine=$1 events=$2: "
  HXF_SERPENTINE=$1 HXF_PCG_EVENTS=$2 python bench.py --no-cpu --steps 30 2>&1 | tail -n 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), 'GDOF/s', round(d['cg_iter']['us'],1), 'us/iter, K1', d['cg_iter']['operator_kernel_us'])"
done
