python -m pytest tests -m gpu -q -x > gpurun_out/g93_pytest.txt 2>&1; tail -n 1 gpurun_out/g93_pytest.txt
for r in 1 2; do
  for v in L0 L3; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/sched_only.py | tail -1; done
  echo -n "L2 "; python tools/sched_only.py | tail -1
done
for r in 1 2 3; do
  for v in L0 L3; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 | tail -1; done
  echo -n "L2 "; python tools/ab_time.py 40 | tail -1
done
for v in L0 L3; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/batch_time.py | tail -1; done
echo -n "L2 "; python tools/batch_time.py | tail -1
