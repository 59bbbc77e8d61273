#!/bin/bash
# A/B of fused-kernel build variants (FWA_B200_LIB selects the .so): per-phase trace and a
# short bench per variant.  Build the variants first, e.g. with -DFWA_POLY_MASK=<m>:
#   libfwa_b200_p<m>.so next to libfwa_b200.so.
for m in "$@"; do
  echo "== variant $m"
  FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$m.so python tools/trace_fused.py 2>&1 | grep -E "loop done|u1 total" | head -3
  FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$m.so python bench.py --steps 30 --warmup 5 --no-batch \
      --no-points --no-equal-window --no-split --no-cpu-baseline 2>&1 | grep -o '"ms_per_step": [0-9.]*'
done
