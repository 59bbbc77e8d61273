python -m pytest tests -m gpu -q -x > gpurun_out/g22_pytest.txt 2>&1; tail -2 gpurun_out/g22_pytest.txt
for r in 1 2; do python tools/ab_time.py 40 2>&1 | tail -1; done
