python -m pytest tests -m gpu -q -x -k "sort or batch or golden or config2 or split" > gpurun_out/g65_pytest.txt 2>&1; tail -n 2 gpurun_out/g65_pytest.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv python tools/sched_batch.py 64 2>/dev/null > gpurun_out/g65_ncu.csv
