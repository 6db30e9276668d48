cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ring2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_overlap_stress.py tests/test_gpu_kernel_modes.py tests/test_gpu_comm.py -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
