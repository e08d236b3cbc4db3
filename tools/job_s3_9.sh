cd /root/repo
ncu -f --set full --import-source on --clock-control none -k regex:accumulate_smem -c 1 -o gpurun_out/c3_accsmem python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 1 --warmup 1 > gpurun_out/ncu_accsmem.log 2>&1
python tools/ncu_summary.py gpurun_out/c3_accsmem.ncu-rep "c3 accumulate_smem" > gpurun_out/s3_accsmem_summary.txt 2>&1
python tools/ncu_hot.py gpurun_out/c3_accsmem.ncu-rep 30 > gpurun_out/s3_accsmem_hot.txt 2>&1
