cd $GRAFT_REPO_ROOT
O=gpurun_out/r02fuse4; mkdir -p $O
for p in 0.5 0.7; do timeout 500 python tools/ab_steps.py 65536,8192,8192 $p 0,65536 3 >> $O/ab.txt 2>&1; done
timeout 400 python tools/ab_steps.py 32768,8192,8192 0.5 0,65536 3 >> $O/ab.txt 2>&1
timeout 400 python tools/ab_steps.py 131072,8192,8192 0.5 0,65536 2 >> $O/ab.txt 2>&1
timeout 400 python tools/ab_steps.py 65536,768,3072 0.5 0,8 4 >> $O/ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_random_layers.py tests/test_gpu_kernel_modes.py -m gpu -q -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
