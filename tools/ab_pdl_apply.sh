timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/apply_stress.py > gpurun_out/apply_stress.log 2>&1; echo rc=$? >> gpurun_out/apply_stress.log
for v in 1 0 1 0; do HXF_PDL_APPLY=$v timeout 300 python bench.py --no-cpu --steps 30 >> gpurun_out/pdla_$v.log 2>&1; done
