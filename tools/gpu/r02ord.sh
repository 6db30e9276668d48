cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ord; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.3" "4096 0.7" "4096 0.9" "2048 0.5" "8192 0.5"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_ord.so $L/var_ord.so:2097152 -r 8 >> $O/ab.txt 2>&1
done
