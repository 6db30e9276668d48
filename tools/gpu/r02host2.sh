cd $GRAFT_REPO_ROOT
O=gpurun_out/r02host2; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python tools/host_probe.py 1024 0.5 > $O/host.txt 2>&1
timeout 300 python tools/gated_probe.py 1024,0.5 1024,0.9 2048,0.5 > $O/gated.jsonl 2>&1
