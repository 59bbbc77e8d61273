python -m pytest tests -m gpu -q > gpurun_out/g76_pytest.txt 2>&1; tail -n 2 gpurun_out/g76_pytest.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/g76_bench.json 2> gpurun_out/g76_bench.err; tail -c 300 gpurun_out/g76_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g76_ref.json 2> gpurun_out/g76_ref.err; tail -c 300 gpurun_out/g76_ref.err
