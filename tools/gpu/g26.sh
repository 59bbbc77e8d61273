python -m pytest tests -m gpu -q -x -k "group_size or fused or golden" > gpurun_out/g26_pytest.txt 2>&1; tail -2 gpurun_out/g26_pytest.txt
python bench.py --steps 10 --warmup 3 --no-batch --no-points --no-equal-window --no-split --no-cpu-baseline > gpurun_out/g26_bench.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/g26_bench.json').read().strip().splitlines()[-1])
print('F60', d['ms_per_step'])
for p in d['config5_sweep']['points']: print(p['frame'], p['G'], round(p['ms_per_frame'],3), round(p['block_tflops'],1))
"
