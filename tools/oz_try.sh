for S in 6 7; do timeout 60 python tools/prof_gemm.py --shape 40000,130,65 --reps 2 --check 1 --opt oz_slices=$S | grep check; done
timeout 60 python tools/prof_gemm.py --shape 40001,130,66 --reps 2 --check 1 --opt oz_slices=7 | grep check
timeout 60 python tools/prof_gemm.py --shape 1000,300,1 --reps 1 --check 1 --opt oz_slices=7 | grep check
for c in c3 c5; do
  for S in 6 7; do timeout 120 python tools/prof_gemm.py --config $c --reps 4 --check 1 --opt oz_slices=$S | tail -2; done
  timeout 120 python tools/prof_gemm.py --config $c --reps 4 --check 1 --opt oz_slices=7 --opt oz_staged=0 | tail -2
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_gemm.py --config c5 --reps 2 --opt oz_slices=7 > gpurun_out/oz_launch_c5.csv 2>&1
timeout 300 ncu -f --set full --import-source on --clock-control none -k regex:oz_gemm -s 1 -c 1 -o gpurun_out/oz_c3 python tools/prof_gemm.py --config c3 --reps 2 --opt oz_slices=7 > /dev/null 2>&1
