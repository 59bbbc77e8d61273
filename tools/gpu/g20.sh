for r in 1 2; do for sp in 103 96 99 110 112; do echo -n "split $sp: "; FWA_B200_SPLIT=$sp python tools/ab_time.py 40 2>&1 | tail -1; done; done
FWA_B200_SPLIT=96 python tools/trace_fused.py 2>&1 | grep -A2 "cta 0:\|cta 1:"
