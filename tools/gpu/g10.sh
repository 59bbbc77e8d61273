for r in 1 2; do
 for v in poly1 poly2; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 30 2>&1 | tail -1; done
 python tools/ab_time.py 30 2>&1 | tail -1
done
for v in poly1 poly2; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/trace_fused.py 2>&1 | grep -A2 "cta 0:\|cta 1:"; done
