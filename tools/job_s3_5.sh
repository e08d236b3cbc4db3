cd /root/repo
for rs in 2 4 6; do for st in 3; do for c in c5 c3; do
  echo "rs=$rs st=$st $(python tools/prof_gemm.py --config $c --reps 4 --opt oz_rs=$rs --opt oz_st=$st 2>&1 | tail -1)"
done; done; done
echo "st=4 rs=2 $(python tools/prof_gemm.py --config c5 --reps 4 --opt oz_rs=2 --opt oz_st=4 2>&1 | tail -1)"
python -m pytest tests -m gpu -q -x -k "ozaki or stage2 or tensor_core or races" 2>&1 | tail -3
