cd $GRAFT_REPO_ROOT
O=gpurun_out/r02j; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernel_modes.py -m gpu -q -x -k "row_pair or wide or masked" > $O/pytest_modes.txt 2>&1; echo "rc=$?" >> $O/pytest_modes.txt
timeout 400 python tools/ab_pairs.py 4096 4096 4096 0.3,0.4,0.5,0.6,0.7 6 > $O/ab_pairs_4096.txt 2>&1
timeout 400 python tools/ab_pairs.py 8192 8192 8192 0.3,0.5 4 > $O/ab_pairs_8192.txt 2>&1
timeout 400 python tools/ab_pairs.py 65536 8192 8192 0.3,0.5 3 > $O/ab_pairs_cfg4.txt 2>&1
