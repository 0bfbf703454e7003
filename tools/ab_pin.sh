for v in 0 24 48 72 0; do HXF_L2_PIN_MB=$v timeout 300 python bench.py --no-cpu --steps 30 > gpurun_out/pin_$v.log 2>&1; cat gpurun_out/pin_$v.log >> gpurun_out/pin_all_$v.log; done
