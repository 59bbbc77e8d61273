python -m pytest tests -m gpu -q -x > gpurun_out/g97_pytest.txt 2>&1; tail -n 1 gpurun_out/g97_pytest.txt
for r in 1 2 3; do
  echo -n "old "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pold.so python tools/sched_only.py | tail -1
  echo -n "new "; python tools/sched_only.py | tail -1
done
for r in 1 2 3; do
  echo -n "old "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pold.so python tools/ab_time.py 40 | tail -1
  echo -n "new "; python tools/ab_time.py 40 | tail -1
done
