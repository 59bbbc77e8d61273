"""Per-kernel SASS opcode histogram of libfwa_b200.so (the evidence that the hot path is
tcgen05 / TMEM / bulk-copy code): cuobjdump -sass, counted per function.

    python tools/sass_hist.py [lib] > profiles/r2_sass.txt
"""
import collections
import os
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "paper_2301_08739_b200",
                                                         "libfwa_b200.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "HMMA", "MUFU", "LDGSTS", "LDSM",
        "LDG", "STG", "LDS", "STS", "SHFL", "BAR", "SYNCS", "FFMA", "HFMA2", "F2FP"]
funcs = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P[T0-9]+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        funcs[cur][m.group(2)] += 1
want = ("k_block_fused", "k_sort_keys", "k_bins_hist", "k_bin_scatter", "k_bin_rank", "k_compact_all", "k_pe_fp16",
        "k_ln1_qkv_tc", "k_outproj_ffn_tc", "k_attention_mma")
print(f"SASS opcode counts per kernel instance ({os.path.basename(lib)}, sm_100a; static instruction counts)")
print(f"{'kernel':70s} " + " ".join(f"{k:>7s}" for k in KEYS))
for f, c in funcs.items():
    try:
        name = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
    except OSError:
        name = f
    if not any(w in name for w in want):
        continue
    short = re.sub(r"fwa_b200::(\(anonymous namespace\)|<unnamed>)::", "", name)
    short = re.sub(r"\(.*\)$", "", short)[:70]
    print(f"{short:70s} " + " ".join(f"{c.get(k, 0):7d}" for k in KEYS))
