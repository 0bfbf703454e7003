for cfg in "bp3 7 20" "bp1 3 40" "bp5 13 12"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:op_ -s 2 -c 1 -o gpurun_out/prof_$1_p$2 python tools/prof_step.py --bp $1 --degree $2 --elems $3 --iters 1 > gpurun_out/prof_$1_p$2.log 2>&1
done
