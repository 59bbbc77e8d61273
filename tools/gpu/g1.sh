set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x > gpurun_out/g1_pytest.txt 2>&1; tail -3 gpurun_out/g1_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.txt 2>&1; tail -2 gpurun_out/g1_smoke.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; tail -c 3000 gpurun_out/g1_bench.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g1_ref.json 2> gpurun_out/g1_ref.err; cat gpurun_out/g1_ref.json
