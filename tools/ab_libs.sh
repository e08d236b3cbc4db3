#!/bin/bash
# Measurement helper (not product code): run a command once per libcgx.so variant
# (build/var/NAME/libcgx.so; "base" = the in-tree library), swapping the in-tree .so.
#   tools/ab_libs.sh "cmd" base v1 v2 ...
cd "$(dirname "$0")/.."
cmd=$1; shift
cp paper_1606_05732_b200/libcgx.so /tmp/libcgx_base.so
for v in "$@"; do
  if [ $v = base ]; then cp /tmp/libcgx_base.so paper_1606_05732_b200/libcgx.so; else cp build/var/$v/libcgx.so paper_1606_05732_b200/libcgx.so; fi
  echo "== $v: $(bash -c "$cmd" 2>&1 | tail -1)"
done
cp /tmp/libcgx_base.so paper_1606_05732_b200/libcgx.so
