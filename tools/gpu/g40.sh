python -m pytest tests -m gpu -q -x -k "repeated or stream or batch or determinism or contract or graph or device" > gpurun_out/g40_pytest.txt 2>&1; tail -2 gpurun_out/g40_pytest.txt
python tools/host_enqueue.py
python bench.py --steps 20 --warmup 5 --no-batch --no-points --no-equal-window --no-split --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['eager']['ms_per_frame'], d['e2e']['ms_per_frame'], d['e2e']['single_frame']['ms_per_frame'])"
