python -m pytest tests -m gpu -q -x -k "fused or golden or config2 or shifted or zero_weights or batch_many or nonfinite or group_size" > gpurun_out/g49_pytest.txt 2>&1; tail -n 2 gpurun_out/g49_pytest.txt
for r in 1 2; do python tools/ab_time.py 40 2>&1 | tail -1; done
