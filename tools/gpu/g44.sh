python -m pytest tests -m gpu -q -x -k "batch or drop or sort or frame_stream or far or compact or cache" > gpurun_out/g44_pytest.txt 2>&1; tail -n 2 gpurun_out/g44_pytest.txt
python tools/sched_batch.py 64 2>&1 | tail -1
python tools/sched_batch.py 1 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g44_sched64.csv python tools/sched_batch.py 64 > /dev/null 2>&1
python tools/launches.py gpurun_out/g44_sched64.csv | tail -12
