# schedule per-kernel split at batch scale + SFU probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/micro/mufu.cu && /tmp/mufu > gpurun_out/g2_mufu.txt 2>&1
cat gpurun_out/g2_mufu.txt
python tools/sched_batch.py 64 > gpurun_out/g2_sched64.txt 2>&1; tail -1 gpurun_out/g2_sched64.txt
python tools/sched_batch.py 1 > gpurun_out/g2_sched1.txt 2>&1; tail -1 gpurun_out/g2_sched1.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g2_sched64.csv python tools/sched_batch.py 64 > /dev/null 2>&1
python tools/launches.py gpurun_out/g2_sched64.csv | tail -30
