python -m pytest tests -m gpu -q -x -k "split or config4" > gpurun_out/g48_pytest.txt 2>&1; tail -n 2 gpurun_out/g48_pytest.txt
python bench.py --steps 10 --warmup 3 --no-sweep --no-batch --no-points --no-equal-window --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config4_split'], d['ms_per_step'])"
