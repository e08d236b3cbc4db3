cd /root/repo
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
B="--no-cpu --no-e2e --no-ablation --steps 20 --warmup 5"
for c in c2 c4; do for v in 1 0 1; do echo "$c small_bulk=$v $(python bench.py --config $c $B --opt small_bulk=$v | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*' | tr '\n' ' ')"; done; done
for c in c2 c4; do python tools/prof_gemm.py --config $c --reps 5 --check 1 2>&1 | tail -1; done
