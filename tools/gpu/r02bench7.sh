cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bench7; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 python -m pytest tests/test_dp_bench.py -q > $O/pytest_dp.txt 2>&1; echo "rc=$?" >> $O/pytest_dp.txt
