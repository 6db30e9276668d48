cd $GRAFT_REPO_ROOT
O=gpurun_out/r03a; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "1024 0.1" "1024 0.5" "1024 0.9" "2048 0.5" "2048 0.9" "4096 0.9" "4096 0.5"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_base.so $L/var_half.so -r 8 >> $O/ab.txt 2>&1
done
for a in "1024 0.5" "1024 0.9" "2048 0.5" "4096 0.9"; do
  timeout 300 python tools/step_parts.py $a 6 >> $O/parts.txt 2>&1
done
