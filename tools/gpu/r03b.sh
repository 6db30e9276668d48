cd $GRAFT_REPO_ROOT
O=gpurun_out/r03b; mkdir -p $O
timeout 600 python tools/gated_probe.py > $O/gated.jsonl 2>&1
