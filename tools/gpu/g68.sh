for r in 1 2; do
for sp in 101 90 96 106 110 117; do
  echo -n "split $sp: "; FWA_B200_SPLIT=$sp python tools/ab_time.py 40 2>&1 | tail -1
done
done
