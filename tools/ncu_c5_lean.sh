set -x
cd /root/repo
O=gpurun_out
B="--no-cpu --no-e2e --no-ablation"
python bench.py --config c5 --steps 2 --warmup 1 $B 2>&1 | tail -1 | cut -c1-600
ncu -f --set full --import-source on --clock-control none -k regex:sketch_csr_lean -s 1 -c 1 \
    -o $O/c5_lean python bench.py --config c5 --steps 2 --warmup 1 $B > $O/ncu_c5.log 2>&1
ls -la $O/c5_lean*
