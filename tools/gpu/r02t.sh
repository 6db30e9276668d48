cd $GRAFT_REPO_ROOT
O=gpurun_out/r02t; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py > $O/bench2.json 2> $O/bench2.err
