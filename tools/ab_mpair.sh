#!/bin/bash
# Measurement helper (not product code): tcgen05 stage 2 with and without M-tile pairs
# (option oz_mpair; oz_cluster 2 = 2 x 2 clusters that also share G's planes) -- accuracy
# against cuBLAS fp64 and time.
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mpair or cluster_and_rings" 2>&1 | tail -1
echo "2x2 $(timeout 120 python tools/prof_gemm.py --config c5 --reps 4 --check 1 2>&1 | tail -1)"
for o in "oz_cluster=2" "oz_cluster=1" "oz_mpair=0" "oz_cluster=2" "oz_cluster=1" "oz_mpair=0"; do
  echo "$o $(timeout 120 python tools/prof_gemm.py --config c5 --reps 4 --opt $o 2>&1 | tail -1 | grep -o 'rep.*')"
done
