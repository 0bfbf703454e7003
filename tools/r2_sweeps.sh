#!/bin/bash
# Round-2 sweeps (profiles/r2_sweep_*): BP5 p=1..15 x 1e5..3e7 DOFs with the
# reference timed beside every point, BP3 / BP6 sweeps, C2 and C4 points.
timeout 2400 python tools/sweep.py --bp bp5 --p 1-15 --sizes 1e5,1e6,1e7,3e7 --cpu --out gpurun_out/r2_sweep_bp5.md --csv gpurun_out/r2_sweep_bp5.csv --records gpurun_out/r2_sweep_bp5_records.jsonl > gpurun_out/r2_sweep_bp5.log 2>&1
timeout 600 python tools/sweep.py --bp bp3 --p 7 --dims 31 --cpu --out gpurun_out/r2_sweep_bp3_c2.md > gpurun_out/r2_sweep_bp3_c2.log 2>&1
timeout 1200 python tools/sweep.py --bp bp6 --p 5-8 --sizes 4.1e7 --cpu --cpu-iters 2 --out gpurun_out/r2_sweep_bp6_c4.md > gpurun_out/r2_sweep_bp6_c4.log 2>&1
timeout 900 python tools/sweep.py --bp bp6 --p 1-15 --sizes 1e7 --out gpurun_out/r2_sweep_bp6.md > gpurun_out/r2_sweep_bp6.log 2>&1
timeout 1200 python tools/sweep.py --bp bp3 --p 1-15 --sizes 1e7 --out gpurun_out/r2_sweep_bp3.md > gpurun_out/r2_sweep_bp3.log 2>&1
for bp in bp1 bp2 bp4; do timeout 600 python tools/sweep.py --bp $bp --p 3,7 --sizes 1e7 --out gpurun_out/r2_sweep_$bp.md > gpurun_out/r2_sweep_$bp.log 2>&1; done
