python -m pytest tests -m gpu -q -x -k "fused or golden or config2 or zero_weights or attention or batch" > gpurun_out/g61_pytest.txt 2>&1; tail -n 2 gpurun_out/g61_pytest.txt
for r in 1 2 3; do
  echo -n "la0 "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pla0.so python tools/ab_time.py 40 2>&1 | tail -1
  echo -n "la1 "; python tools/ab_time.py 40 2>&1 | tail -1
done
