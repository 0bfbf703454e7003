timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/sweep.py --bp bp3 --p 7 --dims 31 > gpurun_out/eo_bp3.log 2>&1
timeout 600 python tools/sweep.py --bp bp5 --p 10-15 --sizes 1e7 > gpurun_out/eo_bp5.log 2>&1
timeout 600 python tools/sweep.py --bp bp3 --p 2,4,10,15 --sizes 1e7 > gpurun_out/eo_bp3b.log 2>&1
timeout 300 python tools/sweep.py --bp bp1 --p 3,7 --sizes 1e7 > gpurun_out/eo_bp1.log 2>&1
