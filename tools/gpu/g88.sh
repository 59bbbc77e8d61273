# grid sizes of the histogram scan (SCAN_G) and the oversize-bin sort (LARGE_G)
for r in 1 2; do
  for v in s16 s48 l16 s16l16; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/sched_only.py | tail -1; done
  echo -n "base "; python tools/sched_only.py | tail -1
done
for v in s16 s16l16; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/batch_time.py | tail -1; done
python tools/batch_time.py | tail -1
