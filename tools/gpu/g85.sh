# k_sort_keys CTAs per spec (partials): F60 schedule alone, F60 frame, 64-frame batch
for r in 1 2; do
  for v in k110 k148 k180 k296; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/sched_only.py | tail -1; done
done
for r in 1 2; do
  for v in k110 k148 k180 k296; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 | tail -1; done
  echo -n "base "; python tools/ab_time.py 40 | tail -1
done
for v in k148 k296; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/batch_time.py | tail -1; done
python tools/batch_time.py | tail -1
