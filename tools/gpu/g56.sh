N="ln1done hs_sync stored_prev lw_done issued table sync_st bK bV bQKV ep_done k_issued bK_leader"
for v in tr trk; do echo "== $v"; FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_p$v.so python tools/trace_detail.py $N | tail -4; done
