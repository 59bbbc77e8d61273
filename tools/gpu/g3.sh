# fresh phase trace + full ncu capture (with source) of the fused block kernel
python tools/trace_fused.py > gpurun_out/g3_trace.txt 2>&1; tail -30 gpurun_out/g3_trace.txt
ncu --set full --import-source on --clock-control none -k regex:k_block_fused -s 9 -c 1 \
    -o gpurun_out/g3_fused python tools/prof_f60.py bf16 2 > gpurun_out/g3_fused.log 2>&1
tail -3 gpurun_out/g3_fused.log
