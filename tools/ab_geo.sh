timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python tools/sweep.py --bp bp5 --p 3-15 --sizes 1e7 > gpurun_out/sw_geo_bp5.log 2>&1
timeout 300 python tools/sweep.py --bp bp3 --p 7 --dims 31 > gpurun_out/sw_geo_bp3.log 2>&1
timeout 600 python tools/sweep.py --bp bp6 --p 5-8 --sizes 4.1e7 > gpurun_out/sw_geo_bp6.log 2>&1
