cd $GRAFT_REPO_ROOT
O=gpurun_out/r02host; mkdir -p $O
timeout 300 python tools/host_probe.py 1024 0.5 > $O/host.txt 2>&1
timeout 300 python tools/host_probe.py 4096 0.5 >> $O/host.txt 2>&1
