python -m pytest tests -m gpu -x -q -k "fused or golden or baseline_configs or determinism or zero_weights or shifted" > gpurun_out/s5_pytest.txt 2>&1
tail -3 gpurun_out/s5_pytest.txt
python bench.py --steps 20 --warmup 5 --no-sweep --no-batch --no-split --no-points --no-equal-window --no-cpu-baseline > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/s5_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['achieved'], d['kernels']['schedule'])"
