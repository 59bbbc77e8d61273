# the headline (plain, graph-replayed) block kernel instance under ncu --set full
ncu --set full --import-source on --clock-control none -k regex:k_block_fused -s 12 -c 1 -o gpurun_out/fused_plain python tools/ab_time.py 2 > gpurun_out/g74_ncu.log 2>&1; tail -n 3 gpurun_out/g74_ncu.log
ls -la gpurun_out/fused_plain.ncu-rep
