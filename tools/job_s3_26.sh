cd /root/repo
B="--no-cpu --no-e2e --no-ablation --steps 3 --warmup 2"
for s in 0 120 100 74 50; do echo "gather_sms=$s $(python bench.py --config c5 $B --opt gather_sms=$s | grep -o '"stage_ms[^}]*')"; done
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k trim 2>&1 | tail -1
