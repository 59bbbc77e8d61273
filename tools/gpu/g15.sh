FWA_TRACE_S5=xwait FWA_TRACE_S6=xsync python tools/trace_fused.py 2>&1 | grep -A2 "cta 0:\|cta 1:\|cta 40:"
