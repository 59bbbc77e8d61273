python -m pytest tests -m gpu -q -x -k "sort or batch or drop or frame_stream or far or compact or cache or golden or config2 or repeated or sparse" > gpurun_out/g46_pytest.txt 2>&1; tail -n 2 gpurun_out/g46_pytest.txt
for r in 1 2 3; do python tools/sched_batch.py 1 2>&1 | tail -1; done
for r in 1 2; do python tools/ab_time.py 40 2>&1 | tail -1; done
