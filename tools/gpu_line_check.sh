timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/sweep.py --bp bp3 --p 7 --dims 31 > gpurun_out/sw_bp3.log 2>&1
timeout 600 python tools/sweep.py --bp bp5 --p 10-15 --sizes 1e7 > gpurun_out/sw_bp5hi.log 2>&1
timeout 600 python tools/sweep.py --bp bp3 --p 1-15 --sizes 1e6 > gpurun_out/sw_bp3all.log 2>&1
timeout 300 python tools/sweep.py --bp bp1 --p 3,7 --sizes 1e7 > gpurun_out/sw_bp1.log 2>&1
