#!/bin/bash
# Build librlb variants that differ only in attention compile-time knobs for
# A/B runs via RLB_LIB=paper_2510_19225_b200/librlb_<tag>.so
#   scripts/build_attn_variants.sh tag:"-DATTN_PAIR_STAGES=3 -DATTN_PAIR_MINB=2" ...
cd "$(dirname "$0")/.."
make -s -j8
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr"
for v in "$@"; do
  tag=${v%%:*}; flags=${v#*:}
  tmp=$(mktemp -d)
  $NV $flags -c paper_2510_19225_b200/csrc/attention.cu -o $tmp/attention.o
  objs="build/engine.o build/gemm.o build/kernels.o build/pull.o build/rowops.o"
  $NV -shared -o paper_2510_19225_b200/librlb_$tag.so $tmp/attention.o $objs -lcudart -ldl
  rm -rf $tmp
  echo built paper_2510_19225_b200/librlb_$tag.so
done
