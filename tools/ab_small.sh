timeout 900 python tools/sweep.py --bp bp5 --p 1-3 --sizes 1e7 > gpurun_out/small_bp5.log 2>&1
timeout 900 python tools/sweep.py --bp bp3 --p 1-3 --sizes 1e7 > gpurun_out/small_bp3.log 2>&1
timeout 900 python tools/sweep.py --bp bp1 --p 1-3 --sizes 1e7 > gpurun_out/small_bp1.log 2>&1
