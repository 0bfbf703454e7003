timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/race_pcg.py > gpurun_out/memcheck_pcg.log 2>&1; echo rc=$? >> gpurun_out/memcheck_pcg.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/race_pcg.py > gpurun_out/racecheck_pcg.log 2>&1; echo rc=$? >> gpurun_out/racecheck_pcg.log
