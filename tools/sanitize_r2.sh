# Round 2: memcheck + racecheck over one apply per operator kernel (incl. the
# even-odd kernel) and over setup + device PCG solves (incl. the fused step kernel)
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/race_cases.py > gpurun_out/r2_memcheck.txt 2>&1; echo rc=$? >> gpurun_out/r2_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/race_cases.py > gpurun_out/r2_racecheck.txt 2>&1; echo rc=$? >> gpurun_out/r2_racecheck.txt
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/race_pcg.py > gpurun_out/r2_memcheck_setup_pcg.txt 2>&1; echo rc=$? >> gpurun_out/r2_memcheck_setup_pcg.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/race_pcg.py > gpurun_out/r2_racecheck_setup_pcg.txt 2>&1; echo rc=$? >> gpurun_out/r2_racecheck_setup_pcg.txt
