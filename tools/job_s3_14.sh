cd /root/repo
for st in 1 0; do for c in c5 c3; do echo "staged=$st $(python tools/prof_gemm.py --config $c --reps 4 --opt oz_staged=$st 2>&1 | tail -1)"; done; done
echo "staged=0 st=4 $(python tools/prof_gemm.py --config c5 --reps 4 --opt oz_staged=0 --opt oz_st=4 2>&1 | tail -1)"
