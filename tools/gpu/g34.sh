timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_tiny.py > gpurun_out/r2_racecheck.txt 2>&1; tail -3 gpurun_out/r2_racecheck.txt
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_tiny.py > gpurun_out/r2_memcheck.txt 2>&1; tail -3 gpurun_out/r2_memcheck.txt
