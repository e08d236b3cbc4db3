#!/bin/bash
# Measurement helper (not product code): rebuild ozgemm.cu with -DOZ_EXP=k (1 = converters
# skip the digits, 2 = no G loads, 3 = no MMAs; results are wrong) and time stage 2 alone.
cd "$(dirname "$0")/../paper_1606_05732_b200/csrc"
for e in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -DOZ_EXP=$e $EXTRA -dc -o ../../build/cgx/ozgemm.o ozgemm.cu
  make -s ../libcgx.so
  for c in c5 c3; do
    echo "OZ_EXP=$e $EXTRA $c: $(cd ../.. && python tools/prof_gemm.py --config $c --reps 4 2>&1 | tail -1)"
  done
done
