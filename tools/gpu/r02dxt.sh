cd $GRAFT_REPO_ROOT
O=gpurun_out/r02dxt; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernel_modes.py -q -k transposed -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
