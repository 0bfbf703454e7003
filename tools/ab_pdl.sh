HXF_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/pdl_tests.log 2>&1; echo rc=$? >> gpurun_out/pdl_tests.log
for v in 1 0 1 0; do HXF_PDL=$v timeout 300 python bench.py --no-cpu --steps 30 >> gpurun_out/pdl_$v.log 2>&1; done
