python bench.py --steps 20 --warmup 5 > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4_ref.json 2> gpurun_out/s4_ref.err
