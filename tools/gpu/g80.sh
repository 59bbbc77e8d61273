# ptxas option variants of the fused kernel's object
for r in 1 2 3; do
  for v in o2 cg ca; do echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 2>&1 | tail -1; done
  echo -n "base "; python tools/ab_time.py 40 2>&1 | tail -1
done
