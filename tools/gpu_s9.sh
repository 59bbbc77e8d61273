python tools/sched_batch.py 64
python tools/sched_batch.py 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s9_sched_batch.csv python tools/sched_batch.py 64 > /dev/null 2>&1
python tools/launches.py gpurun_out/s9_sched_batch.csv | tail -25
