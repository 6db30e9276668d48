cd $GRAFT_REPO_ROOT
O=gpurun_out/r02slab; mkdir -p $O
timeout 600 python tools/slab_probe.py 0.5 > $O/slab_p05.txt 2>&1
timeout 600 python tools/slab_probe.py 0.1 > $O/slab_p01.txt 2>&1
