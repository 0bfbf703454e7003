HXF_DMMA_STAGES=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/gpu_tests_s2.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests_s2.log
for v in 1 2 1 2; do HXF_DMMA_STAGES=$v timeout 300 python bench.py --no-cpu --steps 30 > gpurun_out/stg_$v.log 2>&1; cat gpurun_out/stg_$v.log >> gpurun_out/stg_all_$v.log; done
HXF_DMMA_STAGES=2 timeout 300 python tools/sweep.py --bp bp6 --p 7 --sizes 4.1e7 > gpurun_out/stg_bp6_2.log 2>&1
