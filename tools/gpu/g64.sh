python -m pytest tests -m gpu -q -x -k "positional or golden or config2" > gpurun_out/g64_pytest.txt 2>&1; tail -n 2 gpurun_out/g64_pytest.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:k_pe_fp16 -c 3 --csv python tools/sched_batch.py 64 2>/dev/null | grep k_pe | head -6
