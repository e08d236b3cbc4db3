cd /root/repo
python -m pytest tests/test_csr_atomic.py -m gpu -q -x 2>&1 | tail -3
B="--no-cpu --no-e2e --no-ablation --steps 5 --warmup 3"
for a in 0 1; do python bench.py --config c3 $B --opt csr_acc=$a | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*'; done
for kb in 32 128; do python bench.py --config c3 $B --opt csr_sb_kb=$kb | grep -o '"ms_per_step[^,]*\|"stage_ms[^}]*'; done
python tools/prof_csr_atomic.py 2>&1 | tail -8
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/s3_launches_c3.csv python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 1 --warmup 1 > /dev/null 2>&1
python tools/ncu_csv.py gpurun_out/s3_launches_c3.csv 2>&1 | tail -25
