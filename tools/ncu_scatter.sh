cd /root/repo
timeout 300 ncu -f --set full --import-source on --clock-control none -k regex:scatter_kernel -c 1 -o gpurun_out/c3_scatter python bench.py --config c3 --no-cpu --no-e2e --no-ablation --steps 1 --warmup 1 > gpurun_out/ncu_sc.log 2>&1
ncu -i gpurun_out/c3_scatter.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c3_scatter_src.csv 2>/dev/null
ls -la gpurun_out/c3_scatter*
