cd $GRAFT_REPO_ROOT
O=gpurun_out/r02gs; mkdir -p $O
timeout 600 python tools/isolated_probe.py > $O/iso.jsonl 2> $O/iso.err
