#!/bin/bash
# Measurement helper (not product code): record-path tests, then c3 stage times and the
# record kernels' launch list (duration, DRAM bytes, instructions).
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_csr_atomic.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do timeout 120 python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 10 --warmup 3 | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*' | tr '\n' ' '; echo; done
timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"scatter_kernel|count_kernel|accumulate_kernel" -c 3 --csv --log-file gpurun_out/ab_c3.csv python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 1 --warmup 1 > /dev/null 2>&1
python tools/ncu_csv.py gpurun_out/ab_c3.csv 2>&1 | tail -12
