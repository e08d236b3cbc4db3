#!/bin/bash
# Measurement helper (not product code): stage 2 alone (tools/prof_gemm.py) under option sets.
cd "$(dirname "$0")/.."
make -s -j8 -C paper_1606_05732_b200/csrc
for o in "$@"; do
  for c in c5 c3; do echo "$c $o: $(python tools/prof_gemm.py --config $c --reps 4 $o 2>&1 | tail -1 | cut -d: -f2)"; done
done
