cd $GRAFT_REPO_ROOT
O=gpurun_out/r02n; mkdir -p $O
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> $O/host.txt
timeout 1500 python tools/configs_bench.py --out $O/r02_configs.json > $O/configs.log 2>&1
timeout 900 python tools/fig4_bench.py --out $O/r02_fig4.csv > $O/fig4.log 2>&1
