# memcheck over the GPU parity suite, racecheck (shared-memory hazards) on one
# case per operator kernel
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "apply_vs_oracle or golden" > gpurun_out/memcheck.log 2>&1; echo rc=$? >> gpurun_out/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/race_cases.py > gpurun_out/racecheck.log 2>&1; echo rc=$? >> gpurun_out/racecheck.log
