cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernel_modes.py -m gpu -q -x > $O/pytest_modes.txt 2>&1; echo "rc=$?" >> $O/pytest_modes.txt
timeout 300 python tools/ab_dense.py 4096 8 > $O/ab_dense_4096.txt 2>&1
timeout 400 python tools/ab_dense.py 8192 5 > $O/ab_dense_8192.txt 2>&1
timeout 300 python tools/ab_dense.py 2048 8 > $O/ab_dense_2048.txt 2>&1
