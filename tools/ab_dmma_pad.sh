timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
for v in 1 0; do
  HXF_DMMA_PAD=$v timeout 300 python tools/sweep.py --bp bp5 --p 4-7 --sizes 1e7 > gpurun_out/pad_bp5_$v.log 2>&1
  HXF_DMMA_PAD=$v timeout 300 python tools/sweep.py --bp bp6 --p 5-7 --sizes 4.1e7 > gpurun_out/pad_bp6_$v.log 2>&1
done
