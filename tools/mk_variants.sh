#!/bin/bash
# Build fused-kernel variants as paper_2301_08739_b200/libfwa_b200_p<name>.so (for
# tools/ab_variants.sh): each argument is name=src.cu[:extra nvcc flags]; every other
# object comes from the in-tree build (run `python -c "import __graft_entry__ as g; g.build()"` first).
# OBJ=<file.cu> (default block_fused.cu) names the in-tree source the variant replaces.
set -e
cd "$(dirname "$0")/.."
O=paper_2301_08739_b200/_build
for spec in "$@"; do
  name=${spec%%=*}; rest=${spec#*=}; src=${rest%%:*}; flags=""
  [[ "$rest" == *:* ]] && flags=${rest#*:}
  mkdir -p /tmp/var_$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      -Iinclude -Ipaper_2301_08739_b200/csrc $flags -c $src -o /tmp/var_$name/variant.o
  objs=""
  for f in $O/*.o; do b=$(basename $f); if [ "$b" = "${OBJ:-block_fused.cu}.o" ]; then objs="$objs /tmp/var_$name/variant.o"; else objs="$objs $f"; fi; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2301_08739_b200/libfwa_b200_p$name.so $objs -lcudart -Xlinker -rpath,/usr/local/cuda/lib64
done
