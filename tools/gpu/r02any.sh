cd $GRAFT_REPO_ROOT
O=gpurun_out/r02any; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "2048 0.5" "2048 0.9" "4096 0.5" "4096 0.9" "4096 0.1" "8192 0.5" "1024 0.5"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_cur.so $L/var_any.so -r 8 >> $O/ab.txt 2>&1
done
