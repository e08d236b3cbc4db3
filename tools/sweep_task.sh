#!/bin/bash
# Measurement helper (not product code): step and sketch time vs the dense task size
# (CFG=c2|c4, STEPS=..., KEY=rows_per_task|tail_tasks).
cd "$(dirname "$0")/.."
for r in "$@"; do
  echo "${KEY:-rows_per_task}=$r: $(python bench.py --config ${CFG:-c2} --steps ${STEPS:-400} --warmup 10 --no-cpu --no-e2e --no-ablation --opt ${KEY:-rows_per_task}=$r 2>/dev/null | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["ms_per_step"]*1e3,1), round(j["config"]["stage_ms"]["sketch"]*1e3,1))')"
done
