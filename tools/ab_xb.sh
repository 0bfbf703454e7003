timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
HXF_XBATCH=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/gpu_tests_xb0.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_xb0.log
for v in 1 0 1 0; do HXF_XBATCH=$v timeout 300 python bench.py --no-cpu --steps 30 >> gpurun_out/xb_$v.log 2>&1; done
