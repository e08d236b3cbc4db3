timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/oz_alltests.log 2>&1; echo "rc=$?" >> gpurun_out/oz_alltests.log
for c in c3 c5; do timeout 120 python tools/prof_gemm.py --config $c --reps 4 --check 1 | tail -2; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_gemm.py --config c5 --reps 2 > gpurun_out/oz_launch_c5.csv 2>&1
for c in c3 c5; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-ablation; done
