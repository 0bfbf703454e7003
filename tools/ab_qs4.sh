timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/gpu_tests_qs4.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_qs4.log
HXF_PENCIL=0 timeout 900 python tools/sweep.py --bp bp6 --p 4-6,8,9 --sizes 1e7 > gpurun_out/qs4_line.log 2>&1
timeout 900 python tools/sweep.py --bp bp4 --p 4-7 --sizes 1e7 > gpurun_out/qs4_bp4.log 2>&1
