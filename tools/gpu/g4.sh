# f16 attention: parity subset + A/B against the previous kernel + schedule at batch scale
python -m pytest tests -m gpu -x -q -k "fused or golden or config2 or shifted or zero_weights or determinism or batch or sort or compact or drop" > gpurun_out/g4_pytest.txt 2>&1; tail -3 gpurun_out/g4_pytest.txt
for r in 1 2; do
  for v in base; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 2>&1 | tail -1; done
  python tools/ab_time.py 40 2>&1 | tail -1
done
python tools/sched_batch.py 64 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g4_sched64.csv python tools/sched_batch.py 64 > /dev/null 2>&1
python tools/launches.py gpurun_out/g4_sched64.csv | tail -14
