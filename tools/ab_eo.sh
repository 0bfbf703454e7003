#!/bin/bash
# A/B: even-odd tensor-core kernel (op_dmmaeo.cuh) vs the line / pencil kernels
# it replaces, K1 and CG at ~1e7 DOFs.  Usage: tools/ab_eo.sh [bp5] [8-15] [1e7]
BP=${1:-bp5}; PR=${2:-8-15}; SZ=${3:-1e7}
mkdir -p gpurun_out
for M in 3 0; do
  echo "== HXF_DMMAEO=$M"
  HXF_DMMAEO=$M timeout 900 python tools/sweep.py --bp $BP --p $PR --sizes $SZ --iters 10
done
