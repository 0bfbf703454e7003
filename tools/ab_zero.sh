timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
for v in 0 1 0 1; do HXF_DMMA_MEMSET=$v timeout 300 python bench.py --no-cpu --steps 30 >> gpurun_out/zero_$v.log 2>&1; done
