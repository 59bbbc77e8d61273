FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pnk3.so python -m pytest tests -m gpu -q -x -k "fused or golden or config2 or batch" > gpurun_out/g81_pytest.txt 2>&1; tail -n 2 gpurun_out/g81_pytest.txt
for r in 1 2 3; do
  echo -n "nk3 "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pnk3.so python tools/ab_time.py 40 2>&1 | tail -1
  echo -n "base "; python tools/ab_time.py 40 2>&1 | tail -1
done
