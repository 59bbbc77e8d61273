python -m pytest tests -m gpu -x -q -k "positional or fused or config2" > gpurun_out/s10_pytest.txt 2>&1
tail -2 gpurun_out/s10_pytest.txt
bash tools/gpu_ab.sh chunk peer
python tools/sched_batch.py 64
