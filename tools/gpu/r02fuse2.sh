cd $GRAFT_REPO_ROOT
O=gpurun_out/r02fuse; mkdir -p $O
rm -f $O/ab_fuse_cfg4.txt
for p in 0.3 0.5 0.7; do timeout 500 python tools/ab_steps.py 65536,8192,8192 $p 0,8 3 >> $O/ab_fuse_cfg4.txt 2>&1; done
for p in 0.5; do timeout 500 python tools/ab_steps.py 65536,3072,768 $p 0,8 4 >> $O/ab_fuse_vit.txt 2>&1; done
