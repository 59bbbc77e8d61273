#!/bin/bash
# The ncu evidence summarised under profiles/ (run on ONE GPU under gpurun; numbers
# printed under ncu are never bench values):
#   gpurun --timeout 1500 -- 'bash tools/profile_round.sh'
# (launch list: python tools/launches.py gpurun_out/launches.csv --frame -1)
# then here:  python tools/launches.py gpurun_out/launches.csv > profiles/rN_launches_f60.txt
#             python tools/ncu_summary.py gpurun_out/<rep>.ncu-rep profiles/rN_ncu_<name>.txt ...
OUT=gpurun_out
mkdir -p $OUT
# 1. every launch of the third F60 frame (host API, 8 blocks), warm caches
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
    --log-file $OUT/launches.csv python tools/prof_f60.py bf16 3 > $OUT/launches.log 2>&1
# 2. the fused block kernel (block 1 of the second frame), full set + source
ncu --set full --import-source on --clock-control none -k regex:k_block_fused -s 9 -c 1 \
    -o $OUT/fused python tools/prof_f60.py bf16 2 > $OUT/fused.log 2>&1
# 3. the schedule kernels + PE of the second frame
ncu --set full --clock-control none \
    -k regex:"k_sort_keys|k_bins_hist|k_scan_tiles_dev|k_bin_scatter|k_bin_rank|k_bin_sort_large|k_drop_tables|k_compact_all|k_pe_fp16" \
    -s 9 -c 9 -o $OUT/sched python tools/prof_f60.py bf16 2 > $OUT/sched.log 2>&1
# 4. GPU pillarization of the F60 point cloud
ncu --set full --clock-control none -k regex:"k_cell|k_member|k_pool|k_pillar|k_nonempty" -s 8 -c 8 \
    -o $OUT/pz python tools/prof_pillarize.py 2 > $OUT/pz.log 2>&1
ls -la $OUT
