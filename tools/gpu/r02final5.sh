cd $GRAFT_REPO_ROOT
O=gpurun_out/r02final5; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 1500 python tools/configs_bench.py --out $O/configs.json > $O/configs.log 2>&1
timeout 900 python tools/fig4_bench.py --sizes 1024,2048,4096 --out $O/fig4.csv > $O/fig4.log 2>&1
timeout 300 python tools/gated_probe.py 1024,0.5 1024,0.1 1024,0.9 2048,0.5 > $O/gated.jsonl 2>&1
