cd $GRAFT_REPO_ROOT
O=gpurun_out/r02zd; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.7" "4096 0.3" "4096 0.1" "2048 0.5" "8192 0.5" "8192 0.3" "65536,768,3072 0.5" "65536,3072,768 0.5" "65536,8192,8192 0.5" "65536,8192,8192 0.3"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_base.so $L/var_zc.so $L/var_zl12.so $L/var_zl14.so $L/var_zl16.so $L/var_zl18.so -r 8 >> $O/ab.txt 2>&1
done
