cd $GRAFT_REPO_ROOT
O=gpurun_out/r02smallab2; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "1024 0.5" "1024 0.1" "1024 0.9" "1024,1024,2048 0.5" "512 0.5" "1024,768,3072 0.3" "768 0.5"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_small.so $L/var_smallhalf.so -r 8 >> $O/ab.txt 2>&1
done
