#!/bin/bash
# Measurement helper (not product code): CSR record-path scatter variants (option csr_sc) on
# c3: sketch-phase time and the scatter kernel's ncu duration.
cd "$(dirname "$0")/.."
for v in "$@"; do
  a=$(python tools/prof_csr_atomic.py c3 3 csr_sc=$v | tail -1)
  b=$(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scatter_kernel -c 1 --csv \
      python tools/prof_csr_atomic.py c3 3 csr_sc=$v 2>&1 | grep -v "^==" | tail -1 | awk -F'"' '{print $(NF-1)}')
  echo "csr_sc=$v: $a; scatter $b ns"
done
