cd /root/repo
timeout 300 python -m pytest tests/test_csr_atomic.py -m gpu -q -x 2>&1 | tail -1
for c in c2 c3 c5 c4; do timeout 200 python bench.py --config $c --no-cpu --no-e2e --no-ablation --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), json.dumps(d['roofline']['ceiling']))"; done
