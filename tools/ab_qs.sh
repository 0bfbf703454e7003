timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/pcg_solution_spread.py > gpurun_out/spread.log 2>&1
for v in 1 0; do HXF_XBATCH=$v timeout 300 python bench.py --no-cpu --steps 30 >> gpurun_out/xb2_$v.log 2>&1; done
