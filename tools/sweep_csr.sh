#!/bin/bash
# Measurement helper (not product code): rebuild sketch_csr.cu with CGX_CSR_MINB/CGX_CSR_KW
# variants (min CTAs per SM, item waves in flight) and time the c3/c5 sketch for each.
set -e
cd "$(dirname "$0")/../paper_1606_05732_b200/csrc"
for v in "$@"; do
  set -- $(echo $v | tr ',' ' ')
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -DCGX_CSR_MINB=$1 -DCGX_CSR_KW=$2 -dc -o ../../build/cgx/sketch_csr.o sketch_csr.cu
  make -s ../libcgx.so
  for c in c3 c5; do
    echo "minb=$1 kw=$2 $c: $(cd ../.. && python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-ablation 2>&1 | tail -1 | grep -o 'stage_ms[^,]*')"
  done
done
