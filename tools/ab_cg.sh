#!/bin/bash
# A/B CG-loop options (env toggles), bench CG line
run() {
  echo -n "$1: "
  env $1 python bench.py --no-cpu --steps 30 2>&1 | tail -n 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), 'GDOF/s', round(d['cg_iter']['us'],1), 'us/iter, K1', round(d['cg_iter']['operator_kernel_us'],1), 'apply', round(d['apply']['us'],1))"
}
for cfg in "HXF_PDL=1" "HXF_PDL=0" "HXF_SERPENTINE=0" "HXF_PDL=1"; do run "$cfg"; done
