cd $GRAFT_REPO_ROOT
O=gpurun_out/r02za; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.9" "4096 0.7" "4096 0.3" "2048 0.5" "1024 0.5" "8192 0.5" "65536,8192,8192 0.5"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_base.so $L/var_zc.so $L/var_zc10.so -r 8 >> $O/ab.txt 2>&1
done
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_kernel_modes.py > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
