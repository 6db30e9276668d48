cd $GRAFT_REPO_ROOT
O=gpurun_out/r02zb; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.7" "4096 0.3" "4096 0.1" "2048 0.5" "8192 0.5" "8192 0.1" "65536,768,3072 0.5"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_zc.so $L/var_zc10.so $L/var_n10w4.so $L/var_n6w6.so $L/var_n14w6.so $L/var_n10w8.so $L/var_n20w10.so -r 8 >> $O/ab.txt 2>&1
done
