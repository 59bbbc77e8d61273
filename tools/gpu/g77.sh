N="ln1done bK Kld Kst bV Vld Vst bQKV Qst sync"
GT=1 FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_ptr5.so python tools/trace_detail.py $N | tail -10
