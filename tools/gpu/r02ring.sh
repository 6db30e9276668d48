cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ring; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
L=paper_2411_01238_b200/lib
for a in "1024 0.5" "4096 0.5" "4096 0.9"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_head.so $L/var_ring.so -r 6 >> $O/ab.txt 2>&1
done
