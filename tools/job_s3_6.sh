cd /root/repo
tools/ab_libs.sh "python tools/prof_gemm.py --config c5 --reps 4" base oz1 oz2 oz3 oz5
tools/ab_libs.sh "python tools/prof_gemm.py --config c5 --reps 4 --opt oz_cluster=1" base oz2
