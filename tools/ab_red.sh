timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/red_tests.log 2>&1; echo rc=$? >> gpurun_out/red_tests.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 30 >> gpurun_out/red_bench.log 2>&1; done
timeout 300 python tools/sweep.py --bp bp6 --p 7 --sizes 4.1e7 > gpurun_out/red_bp6.log 2>&1
