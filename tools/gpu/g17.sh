# round-2 evidence: bench line (not under ncu), then the ncu captures
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 400 gpurun_out/r2_bench.json
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
    --log-file $OUT/r2_launches.csv python tools/prof_f60.py bf16 3 > $OUT/r2_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_block_fused -s 9 -c 1 \
    -o $OUT/r2_fused python tools/prof_f60.py bf16 2 > $OUT/r2_fused.log 2>&1
ncu --set full --clock-control none \
    -k regex:"k_sort_keys|k_bins_hist|k_scan_tiles_dev|k_bin_scatter|k_bin_rank|k_bin_sort_large|k_drop_tables|k_compact_all|k_pe_fp16" \
    -s 9 -c 9 -o $OUT/r2_sched python tools/prof_f60.py bf16 2 > $OUT/r2_sched.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/r2_sched64.csv python tools/sched_batch.py 64 > /dev/null 2>&1
python tools/launches.py $OUT/r2_sched64.csv | tail -12
ls -la $OUT | tail -12
