#!/bin/bash
# Measurement helper (not product code): ncu --set full of the c5 stage 2 (M-tile pairs) alone,
# with the SASS-level stall and instruction counts of its barrier waits.
cd "$(dirname "$0")/.."
timeout 120 python tools/prof_gemm.py --config c5 --reps 2 2>&1 | tail -1
timeout 300 ncu -f --set full --import-source on --clock-control none -k regex:oz_gemm -s 1 -c 1 -o gpurun_out/c5_ozmp \
    python tools/prof_gemm.py --config c5 --reps 2 > /dev/null 2>&1
ncu -i gpurun_out/c5_ozmp.ncu-rep --page source --csv --print-source sass > gpurun_out/c5_ozmp_sass.csv 2>/dev/null
rm -f gpurun_out/c5_ozmp.ncu-rep
