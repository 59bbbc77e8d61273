python -m pytest tests -m gpu -q -x > gpurun_out/g11_pytest.txt 2>&1; tail -3 gpurun_out/g11_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m pytest tests -m gpu -q -s -k "baseline_configs" 2>&1 | grep -iE "err|parity" | head -20
for r in 1 2; do FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_pbase.so python tools/ab_time.py 40 2>&1 | tail -1; python tools/ab_time.py 40 2>&1 | tail -1; done
