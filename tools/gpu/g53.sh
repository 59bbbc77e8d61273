python -m pytest tests -m gpu -q -x -k "fp32 or check or golden or config2 or block_forward or oracle" > gpurun_out/g53_pytest.txt 2>&1; tail -n 2 gpurun_out/g53_pytest.txt
python -m pytest tests -m gpu -q -s -k "config2" 2>&1 | grep parity
python tools/check_mode_time.py
