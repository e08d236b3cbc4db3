#!/bin/bash
# Measurement helper (not product code): CSR record-path accumulate variants on c3 (options
# as KEY=VALUE lists, one variant per argument, comma-separated).
cd "$(dirname "$0")/.."
for v in "$@"; do
  opts=$(echo $v | tr ',' ' ')
  a=$(python tools/prof_csr_atomic.py c3 3 $opts | tail -1)
  b=$(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:accumulate_kernel -c 1 --csv \
      python tools/prof_csr_atomic.py c3 3 $opts 2>&1 | grep -v "^==" | tail -1 | awk -F'"' '{print $(NF-1)}')
  echo "$v: $a; accumulate $b ns"
done
