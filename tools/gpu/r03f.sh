cd $GRAFT_REPO_ROOT
O=gpurun_out/r03f; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
L=paper_2411_01238_b200/lib
for a in "1024 0.5" "1024 0.9" "1024 0.1" "2048 0.5" "4096 0.9" "4096 0.5" "4096 0.7" "8192 0.5" "8192 0.9"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_r03.so $L/var_hash.so $L/var_hash.so:524288 -r 8 >> $O/ab.txt 2>&1
done
