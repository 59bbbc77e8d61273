python -m pytest tests -m gpu -q -x -k "far_apart or outlier or sparse_wide or batch or frame_stream or sort or drop or contract" > gpurun_out/g24_pytest.txt 2>&1; tail -3 gpurun_out/g24_pytest.txt
python tools/sched_batch.py 64 2>&1 | tail -1
python tools/sched_batch.py 1 2>&1 | tail -1
