python -m pytest tests -m gpu -q -x > gpurun_out/g12_pytest.txt 2>&1; tail -3 gpurun_out/g12_pytest.txt
for r in 1 2; do for v in base poly1; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 2>&1 | tail -1; done; python tools/ab_time.py 40 2>&1 | tail -1; done
