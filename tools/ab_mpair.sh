#!/bin/bash
# Measurement helper (not product code): tcgen05 stage 2 with and without M-tile pairs
# (option oz_mpair) -- accuracy against cuBLAS fp64 and time, c5 and a c5-like m = 256 shape.
cd "$(dirname "$0")/.."
echo "mpair=1 $(timeout 120 python tools/prof_gemm.py --config c5 --reps 4 --check 1 --opt oz_mpair=1 2>&1 | tail -1)"
for o in "oz_mpair=0" "oz_mpair=1" "oz_mpair=1 --opt oz_rs=2" "oz_mpair=1 --opt oz_rs=3" "oz_mpair=1 --opt oz_st=4 --opt oz_rs=2" "oz_mpair=0"; do
  echo "$o $(timeout 120 python tools/prof_gemm.py --config c5 --reps 4 --opt $o 2>&1 | tail -1 | grep -o 'rep.*')"
done
echo "small: $(timeout 120 python tools/prof_gemm.py --shape 5000,256,70 --reps 2 --check 1 --opt oz_mpair=1 --opt oz_min_z=0 2>&1 | tail -1)"
echo "odd K: $(timeout 120 python tools/prof_gemm.py --shape 100003,512,128 --reps 2 --check 1 --opt oz_mpair=1 2>&1 | tail -1)"
