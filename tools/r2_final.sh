#!/bin/bash
# Round-2 final state: GPU tests, smoke, bench (ours + reference arm)
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.log 2>&1
