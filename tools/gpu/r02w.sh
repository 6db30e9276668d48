cd $GRAFT_REPO_ROOT
O=gpurun_out/r02w; mkdir -p $O
for p in 0.3 0.5 0.7; do timeout 300 python tools/ab_steps.py 4096 $p 0,32 8 >> $O/ab_wide_bwd_4096.txt 2>&1; done
for p in 0.3 0.5; do timeout 400 python tools/ab_steps.py 8192 $p 0,32 4 >> $O/ab_wide_bwd_8192.txt 2>&1; done
