cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
timeout 600 python tools/overhead_probe.py > $O/overhead.jsonl 2> $O/overhead.err
