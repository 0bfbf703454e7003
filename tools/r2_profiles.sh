# Round-2 baseline captures: GPU tests, bench line, launch list, ncu --set full
# of every K1 family at its SURVEY config (for profiles/r2_*).
set -x
python -m pytest tests -m gpu -q -rf -x > gpurun_out/r2_gpu_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r2_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmma -s 30 -c 1 -o gpurun_out/r2_k1_dmma_c3 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_k1_dmma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_pencil -s 2 -c 1 -o gpurun_out/r2_k1_pencil_bp6p8 python tools/prof_step.py --bp bp6 --degree 8 --elems 30 --iters 1 > gpurun_out/r2_k1_pencil.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_pencil -s 2 -c 1 -o gpurun_out/r2_k1_pencil_bp6p5 python tools/prof_step.py --bp bp6 --degree 5 --elems 48 --iters 1 > gpurun_out/r2_k1_pencil5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_dmma -s 2 -c 1 -o gpurun_out/r2_k1_dmmapad_bp6p6 python tools/prof_step.py --bp bp6 --degree 6 --elems 40 --iters 1 > gpurun_out/r2_k1_pad.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_line -s 2 -c 1 -o gpurun_out/r2_k1_line_bp3 python tools/prof_step.py --bp bp3 --degree 7 --elems 31 --iters 1 > gpurun_out/r2_k1_line.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_line -s 2 -c 1 -o gpurun_out/r2_k1_line_bp2 python tools/prof_step.py --bp bp2 --degree 7 --elems 22 --iters 1 > gpurun_out/r2_k1_line_bp2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_line -s 2 -c 1 -o gpurun_out/r2_k1_line_bp4 python tools/prof_step.py --bp bp4 --degree 7 --elems 22 --iters 1 > gpurun_out/r2_k1_line_bp4.log 2>&1
ls -la gpurun_out
