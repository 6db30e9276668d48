cd $GRAFT_REPO_ROOT
O=gpurun_out/r03i; mkdir -p $O
timeout 300 python tools/cold_probe.py 1024 0.5 > $O/cold.txt 2>&1
timeout 300 python tools/cold_probe.py 4096 0.5 >> $O/cold.txt 2>&1
