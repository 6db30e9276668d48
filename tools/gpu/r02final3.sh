cd $GRAFT_REPO_ROOT
O=gpurun_out/r02final3; mkdir -p $O
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> $O/host.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 1500 python tools/configs_bench.py --out $O/configs.json > $O/configs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --profile --steps 3 --warmup 2 --no-cpu > /dev/null 2>&1
