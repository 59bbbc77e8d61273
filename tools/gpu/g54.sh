# what-if timings: PE loads / x-row wait / row stores removed (wrong numerics; bounds only)
for r in 1 2; do
  for v in nope noxw nost noall; do
    echo -n "$v "; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 2>&1 | tail -1
  done
  echo -n "base "; python tools/ab_time.py 40 2>&1 | tail -1
done
FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pnoall.so python tools/trace_fused.py 2>&1 | grep -A3 "cta 0:\|cta 1:"
