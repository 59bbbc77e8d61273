python -m pytest tests -m gpu -q -x -k "sort or batch or golden or config2 or split or frames" > gpurun_out/g66_pytest.txt 2>&1; tail -n 2 gpurun_out/g66_pytest.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_frame_minmax -c 3 --csv python tools/sched_batch.py 64 2>/dev/null | grep duration
