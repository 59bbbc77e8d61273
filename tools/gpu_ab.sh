# usage: bash tools/gpu_ab.sh name1 name2 ... (libfwa_b200_p<name>.so), 3 alternating rounds
for r in 1 2 3; do
  for v in "$@"; do
    FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/ab_time.py 40 2>&1 | tail -1
  done
done
