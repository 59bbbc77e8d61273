FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pt512c74.so python -m pytest tests -m gpu -q -x -k "sort or batch" > gpurun_out/g86_pytest.txt 2>&1; tail -n 1 gpurun_out/g86_pytest.txt
for r in 1 2; do
  for v in t512c74 t512c55 t1024c37 t256c110; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/sched_only.py | tail -1; done
done
for r in 1 2; do
  for v in t512c74 t512c55 t1024c37 t256c110; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 | tail -1; done
done
