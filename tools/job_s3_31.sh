cd /root/repo
python -m pytest tests -m gpu -q -x -k "ozaki or stage2 or tensor_core or races or full_apply or large_z" 2>&1 | tail -1
for cfg in "3 4 4" "3 2 4" "3 3 4" "3 5 2" "3 6 2" "2 6 4" "4 4 2" "2 4 6"; do set -- $cfg
  for c in c5 c3; do echo "st=$1 bst=$2 rs=$3 $(python tools/prof_gemm.py --config $c --reps 4 --opt oz_st=$1 --opt oz_bst=$2 --opt oz_rs=$3 2>&1 | tail -1)"; done
done
