timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/oz_alltests.log 2>&1; echo "rc=$?" >> gpurun_out/oz_alltests.log
for o in "pdl=1" "pdl=0" "pdl=1" "pdl=0"; do timeout 300 python bench.py --steps 600 --warmup 10 --no-cpu --no-e2e --no-ablation --opt $o > gpurun_out/pdl_c2_$o.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/pdl_c2_$o.json')); print('c2 $o', round(d['ms_per_step'],4), d['config']['stage_ms'], d['clocks']['sm_mhz'])"; done
for o in "pdl=1" "pdl=0"; do timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu --no-e2e --no-ablation --opt $o > gpurun_out/pdl_c5_$o.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/pdl_c5_$o.json')); print('c5 $o', round(d['ms_per_step'],4), d['config']['stage_ms'])"; done
