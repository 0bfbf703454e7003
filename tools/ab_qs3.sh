timeout 900 python tools/sweep.py --bp bp3 --p 8,9 --sizes 1e7 > gpurun_out/qs3_bp3.log 2>&1
timeout 900 python tools/sweep.py --bp bp5 --p 9,10 --sizes 1e7 > gpurun_out/qs3_bp5.log 2>&1
