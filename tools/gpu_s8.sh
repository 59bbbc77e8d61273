python -m pytest tests -m gpu -x -q -k "fused or golden or config2 or determinism or zero_weights or shifted or stage" > gpurun_out/s8_pytest.txt 2>&1
tail -2 gpurun_out/s8_pytest.txt
bash tools/gpu_ab.sh r1 b cur
