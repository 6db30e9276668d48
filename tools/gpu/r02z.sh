cd $GRAFT_REPO_ROOT
O=gpurun_out/r02z; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
