for r in 1 2; do for sp in 90 93 96 99 101 103; do echo -n "split $sp: "; FWA_B200_SPLIT=$sp python tools/ab_time.py 40 2>&1 | tail -1; done; done
