cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 > $O/cfg5_g1.json 2> $O/cfg5_g1.err; echo "rc=$?" >> $O/cfg5_g1.err
free -g > $O/free.txt; nproc >> $O/free.txt
