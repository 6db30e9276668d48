cd $GRAFT_REPO_ROOT
O=gpurun_out/r02zc; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.7" "4096 0.3" "4096 0.9" "2048 0.5" "1024 0.5" "8192 0.5" "65536,768,3072 0.5" "65536,3072,768 0.1"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_zc.so $L/var_n14w6.so $L/var_dec6.so $L/var_dec10.so $L/var_dec14.so -r 8 >> $O/ab.txt 2>&1
done
