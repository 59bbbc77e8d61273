python bench.py --steps 20 --warmup 5 --no-batch --no-points --no-equal-window --no-split --no-sweep --no-cpu-baseline 2>gpurun_out/g37.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['eager'], d['stage_timed_ms_per_step'])"
tail -3 gpurun_out/g37.err
