python tools/trace_fused.py 2>&1 | grep -A2 "cta 0:\|cta 1:\|cta 40:\|cta 41:"
