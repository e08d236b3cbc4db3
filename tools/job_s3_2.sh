cd /root/repo
B="--no-cpu --no-e2e --no-ablation --steps 5 --warmup 3"
tools/ab_libs.sh "python bench.py --config c5 $B | grep -o '\"stage_ms[^}]*'" base f128 f256 base f128 > gpurun_out/s3_ab_fetch_c5.txt 2>&1
tools/ab_libs.sh "python bench.py --config c3 --opt csr_mode=1 $B | grep -o '\"stage_ms[^}]*'" base f128 f256 > gpurun_out/s3_ab_fetch_c3.txt 2>&1
tools/ab_libs.sh "python tools/prof_gemm.py --config c5 --reps 4" base oz1 oz3 oz5 base > gpurun_out/s3_ab_oz.txt 2>&1
tools/ab_libs.sh "python tools/prof_gemm.py --config c3 --reps 4" base oz1 oz3 oz5 >> gpurun_out/s3_ab_oz.txt 2>&1
bash tools/ncu_oz.sh > gpurun_out/s3_ncu_oz.txt 2>&1
python tools/ncu_summary.py gpurun_out/c5_oz.ncu-rep "c5 oz_gemm" > gpurun_out/s3_c5_oz_summary.txt 2>&1
python tools/ncu_hot.py gpurun_out/c5_oz.ncu-rep 40 > gpurun_out/s3_c5_oz_hot.txt 2>&1
