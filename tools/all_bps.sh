timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
for bp in bp1 bp2 bp3 bp4 bp5 bp6; do
  timeout 600 python tools/sweep.py --bp $bp --p 3,7 --sizes 1e7 > gpurun_out/allbp_$bp.log 2>&1
done
