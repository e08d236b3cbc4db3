#!/bin/bash
# Measurement helper (not product code): record-path tests, then c3's sketch phase with the
# in-tree library against scatter variants built into build/var/ (tools/build_variant.sh).
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_csr_atomic.py -m gpu -q -x 2>&1 | tail -1
tools/ab_libs.sh "timeout 120 python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 10 --warmup 3 | grep -o '\"stage_ms[^,]*'" base "$@" base "$@"
