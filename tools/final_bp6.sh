timeout 1200 python tools/sweep.py --bp bp6 --p 5-8 --sizes 4.1e7 --cpu --cpu-iters 2 --out gpurun_out/fs_bp6_c4.md > gpurun_out/fs_bp6_c4.log 2>&1
timeout 900 python tools/sweep.py --bp bp6 --p 1-15 --sizes 1e7 --out gpurun_out/fs_bp6.md > gpurun_out/fs_bp6.log 2>&1
