set -x
python -m pytest tests -m gpu -x -q -s -k "baseline_configs or contract or integration" > gpurun_out/s2_pytest_new.txt 2>&1
python -m pytest tests -m gpu -q > gpurun_out/s2_pytest_all.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_tiny.py > gpurun_out/s2_racecheck.txt 2>&1
tail -5 gpurun_out/s2_racecheck.txt
