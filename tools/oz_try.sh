timeout 900 python -m pytest tests -m gpu -x -q -k "csr or ozaki or full_size" > gpurun_out/oz_alltests.log 2>&1; echo "rc=$?" >> gpurun_out/oz_alltests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e --no-ablation > gpurun_out/r01c_launches_c5.csv 2>&1
timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu --no-e2e --no-ablation > gpurun_out/r01c_bench_c5.json 2> gpurun_out/r01c_bench_c5.err
timeout 300 ncu -f --set full --import-source on --clock-control none -k regex:oz_gemm -s 1 -c 1 -o gpurun_out/oz_c5 python tools/prof_gemm.py --config c5 --reps 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/oz_c5.ncu-rep "c5 oz_gemm<7> (tcgen05 kind::i8 stage 2, one launch): ncu --set full --clock-control none" > gpurun_out/r01c_c5_oz_gemm_ncu.txt 2>&1
