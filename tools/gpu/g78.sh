timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_small.py > gpurun_out/g78_race.txt 2>&1; tail -n 2 gpurun_out/g78_race.txt
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_small.py > gpurun_out/g78_mem.txt 2>&1; tail -n 2 gpurun_out/g78_mem.txt
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_small.py > gpurun_out/g78_sync.txt 2>&1; tail -n 2 gpurun_out/g78_sync.txt
