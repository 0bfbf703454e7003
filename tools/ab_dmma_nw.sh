#!/bin/bash
# A/B warps per element of op_dmma_kernel (standalone apply + bench CG line)
for nw in 2 4 8; do
  echo -n "NW=$nw: "; HXF_DMMA_NW=$nw python tools/time_apply.py "$@"
done
