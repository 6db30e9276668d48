cd $GRAFT_REPO_ROOT
O=gpurun_out/r02dxt2; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "4096 0.5" "4096 0.3" "4096 0.7" "4096 0.9" "8192 0.5" "8192 0.3" "65536,8192,8192 0.5" "2048 0.5" "1024 0.5"; do
  timeout 400 python tools/ab_steps_libs.py $a $L/var_dxt.so $L/var_dxt.so:1048576 -r 6 >> $O/ab.txt 2>&1
done
