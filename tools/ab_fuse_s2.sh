#!/bin/bash
# Measurement helper (not product code): the dense sketch with stage 2 folded into its tail
# (option fuse_s2) -- parity tests, then c2 / c4 / c1 steps with and without it.
cd "$(dirname "$0")/.."
timeout 120 python bench.py --config c1 --no-cpu --no-e2e --no-ablation --steps 5 --warmup 3 | grep -o '"ms_per_step[^,]*'
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_races.py -m gpu -q -x -k "dense or countgauss or fused or stage or races or apply" 2>&1 | tail -1
B="--no-cpu --no-e2e --no-ablation --steps 20 --warmup 5"
for c in c2 c4; do for v in 1 0 1 0; do echo "$c fuse_s2=$v $(timeout 120 python bench.py --config $c $B --opt fuse_s2=$v | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*' | tr '\n' ' ')"; done; done
