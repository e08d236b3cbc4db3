#!/bin/bash
# Measurement helper (not product code): re-capture the evidence under profiles/ on a GPU
# box (run under gpurun; writes gpurun_out/prof_*).  Every ncu command runs after the same
# command has exited 0 without ncu.
set -x
cd "$(dirname "$0")/.."
O=gpurun_out
B="--no-cpu --no-e2e --no-ablation"
python bench.py > $O/prof_bench_c2.json 2> $O/prof_bench_c2.err || exit 1
# launch list of a short c2 run
python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/prof_launches_c2.csv \
    python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1
# --set full of the dominant kernels
python bench.py --steps 5 --warmup 3 $B > /dev/null 2>&1 || exit 1
rm -f /tmp/p_*.ncu-rep
ncu -f --set full --import-source on --clock-control none -k regex:sketch_dense_async -s 4 -c 1 -o /tmp/p_c2 \
    python bench.py --steps 5 --warmup 3 $B > /dev/null 2>&1
python tools/ncu_summary.py /tmp/p_c2.ncu-rep "c2 sketch_dense_async" > $O/prof_c2_sketch.txt
for c in c3 c5; do
  python bench.py --config $c --steps 3 --warmup 3 $B > /dev/null 2>&1 || exit 1
  ncu -f --set full --import-source on --clock-control none -k regex:sketch_csr_lean -s 3 -c 1 -o /tmp/p_$c \
      python bench.py --config $c --steps 3 --warmup 3 $B > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/p_$c.ncu-rep "$c sketch_csr_lean" > $O/prof_${c}_csr.txt
done
python tools/prof_gemm.py --config c5 --reps 2 > /dev/null 2>&1 || exit 1
ncu -f --set full --import-source on --clock-control none -k regex:gemm_dmma -s 1 -c 1 -o /tmp/p_g5 \
    python tools/prof_gemm.py --config c5 --reps 2 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/p_g5.ncu-rep "c5 gemm_dmma (one pass over resident G)" > $O/prof_c5_gemm.txt
ls -la $O/prof_*
