timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_partition.py -m gpu -x -q > gpurun_out/gpu_tests_mass.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_mass.log
for bp in bp1 bp2; do timeout 600 python tools/sweep.py --bp $bp --p 3,4,5,7 --sizes 1e7 > gpurun_out/mass_$bp.log 2>&1; done
