python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
python -c "
import json
d=json.loads(open('gpurun_out/r2b_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['e2e']['ms_per_frame'], d['e2e']['pcie_floor_ms_per_frame'], d['roofline']['frac'], d['config3_batch']['ms_per_batch'], d['config4_split']['ms_per_scene'], d['f250_frame']['ms_per_frame'], d['clocks'])
"
