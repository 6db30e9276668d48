cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2>&1
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 > $O/cfg5_g1.json 2> $O/cfg5_g1.err
