cd $GRAFT_REPO_ROOT
O=gpurun_out/r02wa; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.3" "8192 0.5" "65536,8192,8192 0.5" "65536,3072,768 0.5"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_wa3.so $L/var_wa4.so -r 8 >> $O/ab.txt 2>&1
done
