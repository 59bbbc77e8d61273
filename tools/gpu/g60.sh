for r in 1 2 3; do
  echo -n "nostg "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pnostg.so python tools/ab_time.py 40 2>&1 | tail -1
  echo -n "new "; python tools/ab_time.py 40 2>&1 | tail -1
  echo -n "old "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pold.so python tools/ab_time.py 40 2>&1 | tail -1
done
