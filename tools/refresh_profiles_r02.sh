#!/bin/bash
# Measurement helper (not product code): the round-2 evidence under profiles/ (run under
# gpurun; writes gpurun_out/r02_*).  Every ncu command runs after the same command has
# exited 0 without ncu.
set -x
cd "$(dirname "$0")/.."
O=gpurun_out
B="--no-cpu --no-e2e --no-ablation"
python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1
rm -f /tmp/p_*.ncu-rep
python bench.py --steps 5 --warmup 3 $B > /dev/null 2>&1 || exit 1
ncu -f --set full --import-source on --clock-control none -k regex:sketch_dense_async -s 4 -c 1 -o /tmp/p_c2 \
    python bench.py --steps 5 --warmup 3 $B > /dev/null 2>&1
python tools/ncu_summary.py /tmp/p_c2.ncu-rep "c2 sketch_dense_async" > $O/r02_c2_sketch_dense_async_ncu.txt
python bench.py --config c3 --steps 2 --warmup 1 $B > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/r02_launches_c3.csv python bench.py --config c3 --steps 2 --warmup 1 $B > /dev/null 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:"count_kernel|scatter_kernel|accumulate_kernel" -s 3 -c 3 \
    -o /tmp/p_c3 python bench.py --config c3 --steps 2 --warmup 1 $B > /dev/null 2>&1
python tools/ncu_summary.py /tmp/p_c3.ncu-rep "c3 CSR record path (count, scatter, accumulate)" > $O/r02_c3_csr_record_ncu.txt
python bench.py --config c5 --steps 2 --warmup 1 $B > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/r02_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 $B > /dev/null 2>&1
ls -la $O/r02_*
