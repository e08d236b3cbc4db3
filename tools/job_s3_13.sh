cd /root/repo
python -m pytest tests -m gpu -q -x -k "ozaki or stage2 or tensor_core or races or full_apply or large_z" 2>&1 | tail -2
for c in c5 c3; do python tools/prof_gemm.py --config $c --reps 4 --check 1 2>&1 | tail -1; python tools/prof_gemm.py --config $c --reps 4 2>&1 | tail -1; done
python bench.py --config c5 --no-cpu --no-e2e --no-ablation --steps 5 --warmup 3 | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*'
python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 5 --warmup 3 | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*'
