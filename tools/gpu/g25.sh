python -m pytest tests -m gpu -q -x -k "far_apart or outlier or sparse_wide or batch or frame_stream" > gpurun_out/g25_pytest.txt 2>&1; tail -2 gpurun_out/g25_pytest.txt
python tools/sched_batch.py 64 2>&1 | tail -1
