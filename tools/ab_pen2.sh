timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python tools/sweep.py --bp bp6 --p 2,4,5,8,9 --sizes 1e7 > gpurun_out/pen2_bp6.log 2>&1
