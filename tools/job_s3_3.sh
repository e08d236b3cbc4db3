cd /root/repo
for st in 3 4; do for rs in 2 3 4 5; do for cl in 2 1; do
  echo "st=$st rs=$rs cl=$cl c5: $(python tools/prof_gemm.py --config c5 --reps 4 --opt oz_st=$st --opt oz_rs=$rs --opt oz_cluster=$cl 2>&1 | tail -1)"
done; done; done
for st in 3 4; do for rs in 2 4; do
  echo "st=$st rs=$rs c3: $(python tools/prof_gemm.py --config c3 --reps 4 --opt oz_st=$st --opt oz_rs=$rs 2>&1 | tail -1)"
done; done
