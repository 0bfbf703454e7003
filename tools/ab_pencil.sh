timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python tools/sweep.py --bp bp6 --p 2-9 --sizes 1e7 > gpurun_out/pen_bp6.log 2>&1
HXF_PENCIL=0 timeout 900 python tools/sweep.py --bp bp6 --p 2-6,8,9 --sizes 1e7 > gpurun_out/pen_bp6_line.log 2>&1
timeout 600 python tools/sweep.py --bp bp6 --p 5-8 --sizes 4.1e7 > gpurun_out/pen_bp6_c4.log 2>&1
