python -m pytest tests -m gpu -x -q -s -k "split or config4" > gpurun_out/s12_pytest.txt 2>&1
grep -E "parity|passed|failed|Error" gpurun_out/s12_pytest.txt | tail -12
for ex in p2p a2a allgather; do python bench.py --steps 10 --warmup 3 --no-sweep --no-batch --no-points --no-equal-window --no-cpu-baseline --split-exchange $ex 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config4_split'], d['ms_per_step'])"; done
