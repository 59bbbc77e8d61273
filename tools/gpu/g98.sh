FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pr512.so python -m pytest tests -m gpu -q -x -k "sort" > gpurun_out/g98_pytest.txt 2>&1; tail -n 1 gpurun_out/g98_pytest.txt
for r in 1 2 3; do
  for v in r128 r512; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/sched_only.py | tail -1; done
  echo -n "base "; python tools/sched_only.py | tail -1
done
