python -m pytest tests -m gpu -q -x -k "fused or golden or config2 or zero_weights or batch_many or nonfinite or group_size" > gpurun_out/g42_pytest.txt 2>&1; tail -2 gpurun_out/g42_pytest.txt
for r in 1 2 3; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pprev.so python tools/ab_time.py 40 2>&1 | tail -1; python tools/ab_time.py 40 2>&1 | tail -1; done
python tools/trace_fused.py 2>&1 | grep -A1 "cta 0:\|cta 1:"
