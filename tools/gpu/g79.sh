python -m pytest tests -m gpu -q -x -k "fused or golden or config2 or zero_weights or nonfinite or batch or split" > gpurun_out/g79_pytest.txt 2>&1; tail -n 2 gpurun_out/g79_pytest.txt
for r in 1 2 3 4; do
  echo -n "old "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pold.so python tools/ab_time.py 40 2>&1 | tail -1
  echo -n "new "; python tools/ab_time.py 40 2>&1 | tail -1
done
