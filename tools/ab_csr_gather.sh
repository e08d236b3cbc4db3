#!/bin/bash
# Measurement helper (not product code): CSR gather parity tests, then the c5 sketch and the
# c3 gather (csr_mode=1) stage times from the bench.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q -x -k "csr or sparse or fullsize" 2>&1 | tail -3
B="--no-cpu --no-e2e --no-ablation --steps 5 --warmup 3"
python bench.py --config c5 $B 2>&1 | tail -1 | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*'
python bench.py --config c3 --opt csr_mode=1 $B 2>&1 | tail -1 | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*'
