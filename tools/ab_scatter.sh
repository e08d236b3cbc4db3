#!/bin/bash
# Measurement helper (not product code): record-path tests, then c3's sketch phase with the
# in-tree library against the row-loop scatter variant (build/var/rowloop).
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_csr_atomic.py -m gpu -q -x 2>&1 | tail -1
tools/ab_libs.sh "timeout 120 python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 10 --warmup 3 | grep -o '\"stage_ms[^,]*'" base rowloop base rowloop
timeout 200 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"scatter_kernel" -c 1 --csv --log-file gpurun_out/ab_sc.csv python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 1 --warmup 1 > /dev/null 2>&1
python tools/ncu_csv.py gpurun_out/ab_sc.csv 2>&1 | tail -2
