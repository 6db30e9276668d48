cd $GRAFT_REPO_ROOT
O=gpurun_out/r02wave; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernel_modes.py -q -k "wave" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
