cd $GRAFT_REPO_ROOT
O=gpurun_out/r02zh; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.9" "4096 0.8" "4096 0.7" "4096 0.5" "4096 0.3" "2048 0.5" "2048 0.9" "1024 0.5" "8192 0.5" "8192 0.9" "65536,768,3072 0.5" "65536,8192,8192 0.5"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_head.so $L/var_sc14.so $L/var_sc10.so $L/var_sc20.so -r 8 >> $O/ab.txt 2>&1
done
