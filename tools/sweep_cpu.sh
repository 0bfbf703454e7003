timeout 2400 python tools/sweep.py --bp bp5 --p 1-15 --sizes 1e6,1e7 --cpu --out gpurun_out/sweep_bp5_cpu.md > gpurun_out/sweep_bp5_cpu.log 2>&1
timeout 900 python tools/sweep.py --bp bp3 --p 7 --dims 31 --cpu --out gpurun_out/sweep_bp3_cpu.md > gpurun_out/sweep_bp3_cpu.log 2>&1
timeout 1200 python tools/sweep.py --bp bp6 --p 5-8 --sizes 4.1e7 --cpu --cpu-iters 2 --out gpurun_out/sweep_bp6_cpu.md > gpurun_out/sweep_bp6_cpu.log 2>&1
