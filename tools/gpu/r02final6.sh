cd $GRAFT_REPO_ROOT
O=gpurun_out/r02final6; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
