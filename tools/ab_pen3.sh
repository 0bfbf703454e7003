timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/pen3_tests.log 2>&1; echo rc=$? >> gpurun_out/pen3_tests.log
timeout 900 python tools/sweep.py --bp bp6 --p 5,8,9 --sizes 1e7 > gpurun_out/pen3.log 2>&1
timeout 900 python tools/sweep.py --bp bp6 --p 5,8 --sizes 4.1e7 >> gpurun_out/pen3.log 2>&1
