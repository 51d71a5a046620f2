#!/bin/bash
# Build libfreqcache_b200 variants with other backward stream shapes (chunk, unroll, min blocks/SM)
# into tools/ab/bwd_<chunk>_<unroll>_<minblocks>.so, for tools/bwd_bench.py sweeps (FC_LIB_PATH).
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
python -c "import sys; sys.path.insert(0, '$ROOT'); from paper_2208_05321_b200 import build as b; b.build(verbose=False)"
OBJ="$ROOT/build/obj"; mkdir -p "$ROOT/tools/ab" /tmp/bwdvar
for v in "$@"; do
  IFS=_ read c u m <<< "$v"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -I "$ROOT/include" -DFC_BWD_CHUNK=$c -DFC_BWD_UNROLL=$u -DFC_BWD_MINBLOCKS=$m \
    -c "$ROOT/paper_2208_05321_b200/csrc/fc_backward.cu" -o /tmp/bwdvar/fc_backward_$v.o
  objs=""
  for s in fc_api fc_index fc_rows fc_sort fc_engine fc_reorder; do objs="$objs $OBJ/$s.o"; done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
    -o "$ROOT/tools/ab/bwd_$v.so" $objs /tmp/bwdvar/fc_backward_$v.o
  echo "built tools/ab/bwd_$v.so"
done
