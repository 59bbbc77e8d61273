N="ln1done hs park_done(t32) staged(t32) lw_done issued stores_done(t32) sync bK bV bQKV ep_done"
GT=1 FWA_B200_LIB=$PWD/paper_2301_08739_b200/libfwa_b200_ptrn.so python tools/trace_detail.py $N | tail -10
