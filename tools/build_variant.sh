#!/bin/bash
# Measurement helper (not product code): build an A/B variant of libcgx.so into
# build/var/NAME/libcgx.so -- the Makefile's objects with FILES recompiled under extra
# nvcc FLAGS.   tools/build_variant.sh NAME "FLAGS" file.cu [file.cu ...]
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; shift 2
make -s -C paper_1606_05732_b200/csrc
d=build/var/$name; mkdir -p $d; cp build/cgx/*.o $d/
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr"
for f in "$@"; do
  (cd paper_1606_05732_b200/csrc && $NV $flags -dc -o ../../$d/${f%.cu}.o $f)
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $d/libcgx.so $d/*.o -ldl
echo built $d/libcgx.so
