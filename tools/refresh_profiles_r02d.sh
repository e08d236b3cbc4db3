#!/bin/bash
# Measurement helper (not product code): round-2 final evidence (third refresh, after the peer-memory combine) under profiles/ (run under
# gpurun; writes gpurun_out/r02d_*).  Every ncu command runs after the same command has
# exited 0 without ncu.  Bench lines first (full runs incl. cpu_baseline / e2e).
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r02d_pytest_gpu.log 2>&1; tail -1 $O/r02d_pytest_gpu.log
for c in c2 c3 c4 c5 c1; do
  python bench.py --config $c > $O/r02d_bench_$c.json 2> $O/r02d_bench_$c.err || echo "bench $c failed"
done
python bench.py --impl reference > $O/r02d_bench_ref_c2.json 2> $O/r02d_bench_ref_c2.err
B="--no-cpu --no-e2e --no-ablation"
for c in c2 c3 c5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/r02d_launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 $B > /dev/null 2>&1
done
ncu -f --set full --import-source on --clock-control none -k regex:sketch_dense_async -s 4 -c 1 -o $O/r02d_c2_sketch \
    python bench.py --steps 5 --warmup 3 $B > /dev/null 2>&1
python tools/ncu_summary.py $O/r02d_c2_sketch.ncu-rep "c2 sketch_dense_async" > $O/r02d_c2_sketch_dense_async_ncu.txt
ncu -f --set full --import-source on --clock-control none -k regex:"count_kernel|scatter_kernel|accumulate_kernel" -s 3 -c 3 \
    -o $O/r02d_c3_rec python bench.py --config c3 --steps 2 --warmup 1 $B > /dev/null 2>&1
python tools/ncu_summary.py $O/r02d_c3_rec.ncu-rep "c3 CSR record path (count, scatter, accumulate)" > $O/r02d_c3_csr_record_ncu.txt
ncu -f --set full --import-source on --clock-control none -k regex:oz_gemm -s 1 -c 1 -o $O/r02d_c3_oz \
    python bench.py --config c3 --steps 2 --warmup 1 $B > /dev/null 2>&1
python tools/ncu_summary.py $O/r02d_c3_oz.ncu-rep "c3 oz_gemm (tcgen05 stage 2)" > $O/r02d_c3_oz_gemm_ncu.txt
ncu -f --set full --import-source on --clock-control none -k regex:sketch_csr_lean -s 1 -c 1 -o $O/r02d_c5_lean \
    python bench.py --config c5 --steps 2 --warmup 1 $B > /dev/null 2>&1
python tools/ncu_summary.py $O/r02d_c5_lean.ncu-rep "c5 sketch_csr_lean" > $O/r02d_c5_sketch_csr_lean_ncu.txt
ncu -f --set full --import-source on --clock-control none -k regex:oz_gemm -s 1 -c 1 -o $O/r02d_c5_oz \
    python bench.py --config c5 --steps 2 --warmup 1 $B > /dev/null 2>&1
python tools/ncu_summary.py $O/r02d_c5_oz.ncu-rep "c5 oz_gemm (tcgen05 stage 2)" > $O/r02d_c5_oz_gemm_ncu.txt
rm -f $O/*.ncu-rep
ls -la $O/r02d_*
