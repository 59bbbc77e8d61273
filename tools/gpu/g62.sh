N="top pe_ids cpwait sync xs_ld ln1 park park_done"
FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_ptr.so python tools/trace_detail.py $N | tail -6
