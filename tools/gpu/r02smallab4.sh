cd $GRAFT_REPO_ROOT
O=gpurun_out/r02smallab4; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
L=paper_2411_01238_b200/lib
for a in "1024 0.5" "1024 0.9" "512 0.5" "768 0.5" "512 0.1" "768,1536,512 0.5"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_small.so $L/var_smallhalf.so $L/var_smallrule.so -r 8 >> $O/ab.txt 2>&1
done
