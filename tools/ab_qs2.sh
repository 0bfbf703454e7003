timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python tools/sweep.py --bp bp3 --p 1-9 --sizes 1e7 > gpurun_out/qs2_bp3.log 2>&1
timeout 900 python tools/sweep.py --bp bp5 --p 1-6,8,9 --sizes 1e7 > gpurun_out/qs2_bp5.log 2>&1
