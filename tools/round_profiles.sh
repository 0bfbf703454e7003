# launch list of the bench command (per-launch times, cold/serialised) + full
# captures of the top kernels; then the throughput sweeps and the bench line
timeout 400 python bench.py > gpurun_out/bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmma -s 30 -c 1 -o gpurun_out/k1_dmma python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/k1_dmma.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:op_line -s 2 -c 1 -o gpurun_out/k1_line_bp3 python tools/prof_step.py --bp bp3 --degree 7 --elems 31 --iters 1 > gpurun_out/k1_line.log 2>&1
timeout 1500 python tools/sweep.py --bp bp5 --p 1-15 --sizes 1e5,1e6,1e7,3e7 --out gpurun_out/sweep_bp5.md --records gpurun_out/sweep_bp5.jsonl --csv gpurun_out/sweep_bp5.csv > gpurun_out/sweep_bp5.log 2>&1
timeout 400 python tools/sweep.py --bp bp3 --p 7 --dims 31 --out gpurun_out/sweep_bp3.md > gpurun_out/sweep_bp3.log 2>&1
timeout 900 python tools/sweep.py --bp bp3 --p 1-15 --sizes 1e7 --out gpurun_out/sweep_bp3_all.md > gpurun_out/sweep_bp3_all.log 2>&1
timeout 600 python tools/sweep.py --bp bp6 --p 5-8 --sizes 4.1e7 --out gpurun_out/sweep_bp6.md > gpurun_out/sweep_bp6.log 2>&1
