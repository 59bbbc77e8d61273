N="ln1done hs_sync stored_prev lw_done issued table sync_st kvA kvB bQKV ep_done kv_issued"
GT=1 FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_ptrg.so python tools/trace_detail.py $N | tail -10
