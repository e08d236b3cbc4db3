#!/bin/bash
# Measurement helper (not product code): ncu --set full of the c5 tensor-core stage 2 alone.
cd "$(dirname "$0")/.."
python tools/prof_gemm.py --config c5 --reps 2 $@ 2>&1 | tail -1
ncu -f --set full --import-source on --clock-control none -k regex:oz_gemm -s 1 -c 1 -o gpurun_out/c5_oz \
    python tools/prof_gemm.py --config c5 --reps 2 $@ > gpurun_out/ncu_oz.log 2>&1
ls -la gpurun_out/c5_oz.ncu-rep
