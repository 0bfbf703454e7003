set -x
for cfg in "bp3 7 20" "bp6 7 24" "bp5 9 20" "bp5 12 14" "bp5 5 30"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:op_ -s 2 -c 1 -o gpurun_out/prof_$1_p$2 python tools/prof_step.py --bp $1 --degree $2 --elems $3 --iters 1 > gpurun_out/prof_$1_p$2.log 2>&1
done
