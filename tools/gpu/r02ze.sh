cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ze; mkdir -p $O
timeout 1500 python -m pytest -q -x -m gpu tests > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
