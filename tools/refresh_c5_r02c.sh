#!/bin/bash
# Measurement helper (not product code): the c5 line and its stage-2 capture after the M-pair
# kernel became the default (profiles/r02c_*).
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > $O/r02c_pytest.log 2>&1; tail -1 $O/r02c_pytest.log
timeout 600 python bench.py --config c5 > $O/r02c_bench_c5.json 2> $O/r02c_bench_c5.err
timeout 300 ncu -f --set full --import-source on --clock-control none -k regex:oz_gemm -s 1 -c 1 -o $O/r02c_c5_oz \
    python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e --no-ablation > /dev/null 2>&1
python tools/ncu_summary.py $O/r02c_c5_oz.ncu-rep "c5 oz_gemm<7, MP> (tcgen05 stage 2, M-tile pairs)" > $O/r02c_c5_oz_gemm_ncu.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/r02c_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e --no-ablation > /dev/null 2>&1
rm -f $O/*.ncu-rep
