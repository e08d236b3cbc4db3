#!/bin/bash
# Measurement helper (not product code): the bench configs with libcgx built with -dc
# (relocatable device code, the Makefile's) and without (whole-program per file,
# build/nodc/libcgx.so) -- same sources.
cd "$(dirname "$0")/.."
B="--steps 10 --warmup 3 --no-cpu --no-e2e --no-ablation"
cp paper_1606_05732_b200/libcgx.so /tmp/libcgx_dc.so
for v in dc nodc dc nodc; do
  if [ $v = nodc ]; then cp build/nodc/libcgx.so paper_1606_05732_b200/libcgx.so; else cp /tmp/libcgx_dc.so paper_1606_05732_b200/libcgx.so; fi
  for c in c2 c3 c4 c5; do
    echo "$v $c: $(python bench.py --config $c $B 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["ms_per_step"],4), {k: round(v,4) for k,v in j["config"]["stage_ms"].items() if isinstance(v,float)})')"
  done
done
cp /tmp/libcgx_dc.so paper_1606_05732_b200/libcgx.so
