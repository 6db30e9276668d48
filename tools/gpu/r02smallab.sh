cd $GRAFT_REPO_ROOT
O=gpurun_out/r02smallab; mkdir -p $O
L=paper_2411_01238_b200/lib
for a in "1024 0.5" "1024 0.1" "1024 0.9" "1024,1024,2048 0.5" "512 0.5" "1024,768,3072 0.3"; do
  timeout 300 python tools/ab_steps_libs.py $a $L/var_small.so $L/var_small.so:2097152 -r 8 >> $O/ab.txt 2>&1
done
timeout 300 python tools/cold_probe.py 1024 0.5 > $O/cold_hash.txt 2>&1
SD_TUNING=2097152 timeout 300 python tools/cold_probe.py 1024 0.5 > $O/cold_list.txt 2>&1
timeout 300 python tools/gated_probe.py 1024,0.5 1024,0.1 1024,0.9 > $O/gated_hash.jsonl 2>&1
SD_TUNING=2097152 timeout 300 python tools/gated_probe.py 1024,0.5 > $O/gated_list.jsonl 2>&1
