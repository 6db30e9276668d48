cd $GRAFT_REPO_ROOT
O=gpurun_out/r03k; mkdir -p $O
cp paper_2411_01238_b200/lib/var_gflag.so paper_2411_01238_b200/lib/libsparsedrop_b200.so
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
L=paper_2411_01238_b200/lib
for a in "1024 0.5" "1024 0.1" "1024 0.9" "2048 0.5" "4096 0.5" "4096 0.9" "8192 0.5"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_head.so $L/var_gflag.so $L/var_gflag.so:131072 -r 8 >> $O/ab.txt 2>&1
done
