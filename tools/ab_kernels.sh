#!/bin/bash
# A/B the collocated operator kernels (standalone apply, CUDA events)
for k in dmma pencil generic; do
  echo -n "$k: "; HXF_OP_KERNEL=$k python tools/time_apply.py "$@"
done
