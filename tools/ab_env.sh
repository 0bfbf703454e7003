#!/bin/bash
# A/B of one env knob on the C3 bench step: tools/ab_env.sh VAR "v1 v2 ..." [reps]
VAR=$1; VALS=$2; REPS=${3:-2}
for r in $(seq $REPS); do for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --no-cpu --steps 30 > gpurun_out/ab_env.log 2>&1
  python - "$VAR=$v" <<'PY'
import json, sys
l = [x for x in open("gpurun_out/ab_env.log") if x.startswith("{")]
d = json.loads(l[-1])
print(sys.argv[1], round(d["value"], 3), round(d["cg_iter"]["us"], 2), round(d["cg_iter"]["operator_kernel_us"], 2),
      round(d["roofline"]["frac"], 4))
PY
done; done
