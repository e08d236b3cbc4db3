cd /root/repo
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stage2 or small or gemm or countgauss" 2>&1 | tail -2
B="--no-cpu --no-e2e --no-ablation --steps 20 --warmup 5"
for c in c2 c4; do for v in 1 0 1; do echo "$c small_bulk=$v $(timeout 120 python bench.py --config $c $B --opt small_bulk=$v | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*' | tr '\n' ' ')"; done; done
for c in c2 c4; do timeout 120 python tools/prof_gemm.py --config $c --reps 5 --check 1 2>&1 | tail -1; done
