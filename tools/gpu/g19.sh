python -m pytest tests -m gpu -q -x -k "stage or contract or frame_stream or integration" > gpurun_out/g19_pytest.txt 2>&1; tail -2 gpurun_out/g19_pytest.txt
for r in 1 2; do
python bench.py --steps 20 --warmup 5 --no-batch --no-points --no-equal-window --no-split --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('value', d['ms_per_step'], 'stream', e['ms_per_frame'], 'floor', e['pcie_floor_ms_per_frame'], 'single', e['single_frame']['ms_per_frame'])"
done
