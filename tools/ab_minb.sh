timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/gpu_tests_m5.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests_m5.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 30 >> gpurun_out/minb5.log 2>&1; done
timeout 300 python tools/sweep.py --bp bp6 --p 6,7 --sizes 4.1e7 > gpurun_out/minb5_bp6.log 2>&1
timeout 300 python tools/sweep.py --bp bp5 --p 7 --sizes 1e7,3e7 > gpurun_out/minb5_bp5.log 2>&1
