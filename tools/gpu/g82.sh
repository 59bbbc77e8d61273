python -m pytest tests -m gpu -q -x -k "frames or stream or e2e or repeated" > gpurun_out/g82_pytest.txt 2>&1; tail -n 2 gpurun_out/g82_pytest.txt
A="--no-split --no-points --no-equal-window --no-sweep --no-batch --no-cpu-baseline"
for r in 1 2 3; do
  FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pold.so python bench.py $A 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('old e2e', round(e['ms_per_frame'],4), 'floor', round(e['pcie_floor_ms_per_frame'],4))"
  python bench.py $A 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('new e2e', round(e['ms_per_frame'],4), 'floor', round(e['pcie_floor_ms_per_frame'],4))"
done
