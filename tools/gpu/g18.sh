for r in 1 2; do
python bench.py --steps 20 --warmup 5 --no-batch --no-points --no-equal-window --no-split --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('stage on ', d['ms_per_step'], e['ms_per_frame'], e['pcie_floor_ms_per_frame'], e['single_frame']['ms_per_frame'])"
FWA_B200_NO_STAGE_TIMES=1 python bench.py --steps 20 --warmup 5 --no-batch --no-points --no-equal-window --no-split --no-sweep --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('stage off', d['ms_per_step'], e['ms_per_frame'], e['pcie_floor_ms_per_frame'], e['single_frame']['ms_per_frame'])"
done
