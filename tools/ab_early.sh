timeout 900 python tools/sweep.py --bp bp5 --p 10-15 --sizes 1e7 > gpurun_out/early_bp5.log 2>&1
timeout 900 python tools/sweep.py --bp bp3 --p 9-15 --sizes 1e7 > gpurun_out/early_bp3.log 2>&1
