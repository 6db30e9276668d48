cd $GRAFT_REPO_ROOT
O=gpurun_out/r02smallab3; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "1024 0.5" "1024 0.1" "1024 0.9" "512 0.5" "768 0.5" "1024,1024,2048 0.5"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_smallhalf.so $L/var_smallall.so -r 8 >> $O/ab.txt 2>&1
done
timeout 300 python tools/cold_probe.py 1024 0.5 > $O/cold.txt 2>&1
