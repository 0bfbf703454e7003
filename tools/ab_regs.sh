timeout 900 python tools/sweep.py --bp bp3 --p 1-15 --sizes 1e7 > gpurun_out/regs_bp3.log 2>&1
timeout 900 python tools/sweep.py --bp bp5 --p 1-6,8-15 --sizes 1e7 > gpurun_out/regs_bp5.log 2>&1
timeout 300 python tools/sweep.py --bp bp6 --p 3,10 --sizes 1e7 > gpurun_out/regs_bp6.log 2>&1
