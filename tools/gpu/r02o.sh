cd $GRAFT_REPO_ROOT
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernel_modes.py tests/test_gpu_parity.py tests/test_gpu_large_configs.py -m gpu -q -x > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 400 python tools/ab_libs.py tools/ablibs/lib_before.so paper_2411_01238_b200/lib/libsparsedrop_b200.so 4096 0.5 8 > $O/ab_4096_p05.txt 2>&1
timeout 400 python tools/ab_libs.py tools/ablibs/lib_before.so paper_2411_01238_b200/lib/libsparsedrop_b200.so 8192 0.5 4 > $O/ab_8192_p05.txt 2>&1
timeout 300 python tools/ab_libs.py tools/ablibs/lib_before.so paper_2411_01238_b200/lib/libsparsedrop_b200.so 4096 0.9 8 > $O/ab_4096_p09.txt 2>&1
