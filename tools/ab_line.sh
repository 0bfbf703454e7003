timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/sweep.py --bp bp3 --p 7 --dims 31 > gpurun_out/ab_bp3_0.log 2>&1
timeout 300 python tools/sweep.py --bp bp5 --p 10-15 --sizes 1e7 > gpurun_out/ab_bp5_0.log 2>&1
timeout 300 python tools/sweep.py --bp bp6 --p 8 --sizes 4.1e7 > gpurun_out/ab_bp6_0.log 2>&1
