cd $GRAFT_REPO_ROOT
O=gpurun_out/r02fuse; mkdir -p $O
for p in 0.3 0.5 0.7; do timeout 300 python tools/ab_steps.py 4096 $p 0,8 8 >> $O/ab_fuse_4096.txt 2>&1; done
for p in 0.3 0.5 0.7; do timeout 400 python tools/ab_steps.py 8192 $p 0,8 4 >> $O/ab_fuse_8192.txt 2>&1; done
for p in 0.3 0.5; do timeout 400 python tools/ab_tuning.py 65536,8192,8192 $p 0,8 3 >> $O/ab_fuse_cfg4.txt 2>&1; done
