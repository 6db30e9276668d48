cd $GRAFT_REPO_ROOT
O=gpurun_out/r03e; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.9" "4096 0.8" "8192 0.9" "2048 0.9" "1024 0.9" "1024 0.1" "2048 0.5"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_base.so $L/var_r03.so $L/var_r03.so:262144 -r 8 >> $O/ab.txt 2>&1
done
