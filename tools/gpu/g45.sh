python -m pytest tests -m gpu -q > gpurun_out/r2f_pytest.txt 2>&1; tail -n 3 gpurun_out/r2f_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
python -c "
import json
d=json.loads(open('gpurun_out/r2f_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['eager']['ms_per_frame'], d['e2e']['ms_per_frame'], d['e2e']['pcie_floor_ms_per_frame'], d['roofline']['frac'], d['config3_batch']['ms_per_batch'], d['config4_split']['ms_per_scene'], d['clocks'])"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2f_ref.json 2>/dev/null; tail -c 300 gpurun_out/r2f_ref.json
