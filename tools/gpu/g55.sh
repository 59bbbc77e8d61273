FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_ptr.so python tools/trace_detail.py ln1done hs_sync stored_prev lw_done issued table sync_st bK bV bQKV ep_done
