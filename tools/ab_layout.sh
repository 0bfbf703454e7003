timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_partition.py -m gpu -x -q > gpurun_out/layout_tests.log 2>&1; echo rc=$? >> gpurun_out/layout_tests.log
timeout 900 python tools/sweep.py --bp bp3 --p 4-15 --sizes 1e7 > gpurun_out/layout_bp3.log 2>&1
timeout 900 python tools/sweep.py --bp bp5 --p 5,6,9,13 --sizes 1e7 > gpurun_out/layout_bp5.log 2>&1
