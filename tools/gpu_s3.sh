python -m pytest tests -m gpu -x -q -k "far_apart or outlier or sparse_wide or batch or contract or integration or sort" > gpurun_out/s3_pytest.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_tiny.py > gpurun_out/s3_racecheck.txt 2>&1
tail -3 gpurun_out/s3_racecheck.txt
