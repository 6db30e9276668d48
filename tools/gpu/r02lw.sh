cd $GRAFT_REPO_ROOT
O=gpurun_out/r02lw; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.3" "8192 0.5" "65536,8192,8192 0.5" "65536,3072,768 0.5" "2048 0.5"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_lw4.so $L/var_lw8.so $L/var_lw12.so $L/var_lw16.so -r 6 >> $O/ab.txt 2>&1
done
