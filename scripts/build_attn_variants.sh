#!/bin/bash
# Build librlb variants that differ only in the decode attention's pipeline
# depth / CTAs per SM (compile-time ATTN_STAGES / ATTN_MINB) for A/B runs via
# RLB_LIB=paper_2510_19225_b200/librlb_<tag>.so
cd "$(dirname "$0")/.."
make -s -j8
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr"
for v in "$@"; do   # v = STAGES:MINB
  s=${v%%:*}; b=${v##*:}; tag="s${s}b${b}"
  $NV -DATTN_STAGES=$s -DATTN_MINB=$b -c paper_2510_19225_b200/csrc/attention.cu -o build/attention_$tag.o
  objs=$(ls build/*.o | grep -v "attention" | tr '\n' ' ')
  $NV -shared -o paper_2510_19225_b200/librlb_$tag.so build/attention_$tag.o $objs -lcudart -ldl
  echo built paper_2510_19225_b200/librlb_$tag.so
done
