# FMA-pipe exponential share: 2 = tiles 3,7 (2/9, default); 3 = tiles 2,5,8; 4 = tiles 1,4,7 (3/9); 5 = tiles 3,6
for r in 1 2 3; do
  for v in poly3 poly4 poly5; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 2>&1 | tail -1; done
  echo -n "base "; python tools/ab_time.py 40 2>&1 | tail -1
done
