python tools/trace_fused.py > gpurun_out/r2_trace.txt 2>&1; head -30 gpurun_out/r2_trace.txt
ncu --set full --import-source on --clock-control none -k regex:k_block_fused -s 9 -c 1 \
    -o gpurun_out/r2c_fused python tools/prof_f60.py bf16 2 > gpurun_out/r2c_fused.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
    --log-file gpurun_out/r2c_launches.csv python tools/prof_f60.py bf16 3 > /dev/null 2>&1
