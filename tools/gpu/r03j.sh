cd $GRAFT_REPO_ROOT
O=gpurun_out/r03j; mkdir -p $O
timeout 600 python tools/gated_probe.py 1024,0.5 1024,0.1 2048,0.5 4096,0.5 > $O/gated.jsonl 2>&1
