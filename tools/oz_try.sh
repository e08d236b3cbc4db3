for S in 6 7; do for o in "oz_dbg=0" "oz_dbg=4"; do
for r in 1 2 3; do timeout 60 python tools/prof_gemm.py --shape 20011,96,300 --reps 3 --check 1 --opt oz_min_z=0 --opt oz_slices=$S --opt $o | grep check; done
done; done
for c in c3 c5; do for o in "oz_dbg=0" "oz_dbg=4"; do timeout 120 python tools/prof_gemm.py --config $c --reps 4 --check 1 --opt $o | tail -2; done; done
