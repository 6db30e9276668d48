cd $GRAFT_REPO_ROOT
O=gpurun_out/r02dxt3; mkdir -p $O
timeout 300 python tools/dx_kernels.py 4096 0.3 0.5 0.7 > $O/dx.txt 2>&1
timeout 300 python tools/dx_kernels.py 8192 0.5 >> $O/dx.txt 2>&1
timeout 300 python tools/dx_kernels.py 65536,8192,8192 0.5 >> $O/dx.txt 2>&1
