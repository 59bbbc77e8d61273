python -m pytest tests -m gpu -x -q -k "fused or golden or config2 or shifted or zero_weights or determinism or baseline_configs" > gpurun_out/g5_pytest.txt 2>&1; tail -3 gpurun_out/g5_pytest.txt
grep -E "err|parity" gpurun_out/g5_pytest.txt | head
for r in 1 2; do
  FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pbase.so python tools/ab_time.py 40 2>&1 | tail -1
  python tools/ab_time.py 40 2>&1 | tail -1
done
python tools/trace_fused.py > gpurun_out/g5_trace.txt 2>&1; grep -A3 "cta 0:\|cta 1:" gpurun_out/g5_trace.txt
